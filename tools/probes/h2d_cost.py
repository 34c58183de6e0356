# host cost of uploading one pinned frame (1280x720 RGBA, 3.7 MB): .to() vs empty+copy_ vs
# empty + cudaMemcpyAsync (cuda-python), all on a side stream, no synchronisation in the loop
import time, torch
from cuda.bindings import runtime as rt
x = torch.randint(0, 255, (720, 1280, 4), dtype=torch.uint8).pin_memory()
s = torch.cuda.Stream()
n = 200
def bench(name, f):
    for _ in range(10): f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): f()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"{name}: {1e6 * (t1 - t0) / n:.1f} us/call")
def f_to():
    with torch.cuda.stream(s):
        d = x.to("cuda", non_blocking=True)
def f_copy():
    with torch.cuda.stream(s):
        d = torch.empty(x.shape, dtype=x.dtype, device="cuda")
        d.copy_(x, non_blocking=True)
buf = torch.empty(x.shape, dtype=x.dtype, device="cuda")
def f_copy_pre():
    with torch.cuda.stream(s):
        buf.copy_(x, non_blocking=True)
def f_rt():
    d = torch.empty(x.shape, dtype=x.dtype, device="cuda")
    rt.cudaMemcpyAsync(d.data_ptr(), x.data_ptr(), x.numel(), rt.cudaMemcpyKind.cudaMemcpyHostToDevice, s.cuda_stream)
def f_rt_pre():
    rt.cudaMemcpyAsync(buf.data_ptr(), x.data_ptr(), x.numel(), rt.cudaMemcpyKind.cudaMemcpyHostToDevice, s.cuda_stream)
def f_ev():
    e = torch.cuda.Event(); e.record(s)
for name, f in (("to", f_to), ("empty+copy_", f_copy), ("prealloc copy_", f_copy_pre), ("empty+cudart", f_rt),
                ("prealloc cudart", f_rt_pre), ("event", f_ev)):
    bench(name, f)
