#!/bin/bash
# scratch GPU session script (gpurun)
python -m pytest tests/test_gpu_render_refine.py tests/test_gpu_edges.py tests/test_gpu_sortfree.py tests/test_gpu_pipeline.py -m gpu -x -q 2>&1 | tail -3
bash tools/ab.sh "--steps 20 --warmup 5 --no-cpu-baseline --no-e2e" base pdl > gpurun_out/ab.log 2>&1
cat gpurun_out/ab.log
