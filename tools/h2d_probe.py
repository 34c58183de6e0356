"""Diagnostic: host->device upload cost of one frame per dtype (pinned)."""
import time

import torch

for dt in (torch.int16, torch.uint16, torch.uint8):
    n = 921600 * (4 if dt == torch.uint8 else 1)
    x = torch.zeros(n, dtype=dt).pin_memory()
    torch.cuda.synchronize()
    for trial in range(2):
        t0 = time.time()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for k in range(10):
            a = x.to("cuda", non_blocking=True)
        e1.record()
        th = time.time() - t0
        torch.cuda.synchronize()
        print(dt, "10 uploads: device ms %.3f host ms %.3f" % (e0.elapsed_time(e1), th * 1e3))
    x16 = x.view(torch.int16) if dt == torch.uint16 else None
    if x16 is not None:
        t0 = time.time()
        for k in range(10):
            a = x16.to("cuda", non_blocking=True).view(torch.uint16)
        print("uint16 via int16 view: host ms %.3f" % ((time.time() - t0) * 1e3))
