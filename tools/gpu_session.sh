#!/bin/bash
# scratch GPU session script (gpurun): parity tests touched this round, smoke, probes, bench variants
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests/test_gpu_fuse_raycast.py tests/test_gpu_chain.py tests/test_gpu_edges.py -m gpu -x -q -s 2>&1 | tail -40 > gpurun_out/t1.log
python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke.log 2>&1
./tools/probes/ffma2 > gpurun_out/ffma2.log 2>&1
python tools/raycast_stats.py > gpurun_out/raystats.log 2>&1
for g in workspace none scene; do
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline --dense-grid $g > gpurun_out/bench_$g.json 2> gpurun_out/bench_$g.err
done
cat gpurun_out/t1.log gpurun_out/smoke.log gpurun_out/ffma2.log gpurun_out/raystats.log
for g in workspace none scene; do python -c "import json;d=json.load(open('gpurun_out/bench_$g.json'));print('$g',d['value'],d['e2e']['value'],{k:v['ms_per_step'] for k,v in d['kernels'].items()})"; tail -3 gpurun_out/bench_$g.err; done
