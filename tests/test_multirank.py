"""Multi-rank host logic of bench.py on CPU (gloo, world_size 2): every rank maps an independent
sequence, the job time is the max over ranks, the job rate counts all ranks' frames, and the
reference arm runs on rank 0 only (replicas, no data-path collective)."""
import os
import subprocess
import sys

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    cfg = bench.rank_config("cfg4", rank, world)
    ms = 100.0 + 50.0 * rank
    m = bench.max_over_ranks(ms, "cpu")
    q.put((rank, cfg.seed, m, bench.job_rate(200, world, m)))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_independent_sequences_and_max_time():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 2000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, s0, m0, v0), (r1, s1, m1, v1) = out
    assert s0 != s1                     # independent rooms / trajectories per rank
    assert m0 == m1 == 150.0            # the slowest rank's time
    assert v0 == v1 == pytest.approx(2 * 200 / 0.150)  # all ranks' frames / max time


def test_single_rank_uses_the_config_seed():
    import bench
    import gps_synth as S
    assert bench.rank_config("cfg4", 0, 1).seed == S.get_config("cfg4").seed
    assert bench.max_over_ranks(12.5, "cpu") == 12.5


def test_reference_arm_only_on_rank_0():
    """Under torchrun the reference (oracle) arm runs on rank 0; other ranks exit 0 silently."""
    env = dict(os.environ, WORLD_SIZE="2", RANK="1", LOCAL_RANK="1")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1"],
                       env=env, capture_output=True, text=True, timeout=300)
    assert p.returncode == 0 and p.stdout.strip() == ""


def test_reference_arm_prints_the_contract_line():
    """bench.py --impl reference (the oracle arm) on the small cfg1 case: one JSON line with the
    reference keys, zero host<->device bytes and a positive rate."""
    import json
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "cfg1",
                        "--steps", "1"], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr
    d = json.loads(p.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "frames/s"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["config"]["workload"].startswith("cfg1")
