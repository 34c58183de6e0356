#!/bin/bash
# scratch GPU session script (gpurun)
python -m pytest tests/test_gpu_render_refine.py tests/test_gpu_chain.py tests/test_gpu_edges.py -m gpu -x -q 2>&1 | tail -4 > gpurun_out/t1.log
cat gpurun_out/t1.log
bash tools/ab.sh "--steps 20 --warmup 5 --no-cpu-baseline" base gbwd > gpurun_out/ab.log 2>&1
cat gpurun_out/ab.log
