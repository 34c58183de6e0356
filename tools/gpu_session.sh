#!/bin/bash
# scratch GPU session script (gpurun)
python -m pytest tests/test_gpu_render_refine.py tests/test_gpu_edges.py tests/test_gpu_sortfree.py tests/test_gpu_chain.py tests/test_gpu_pipeline.py -m gpu -x -q -s 2>&1 | grep -v "^    " | tail -25 > gpurun_out/t1.log
cat gpurun_out/t1.log
bash tools/ab.sh "--steps 20 --warmup 5 --history 2500 --no-cpu-baseline" long split > gpurun_out/ab.log 2>&1
bash tools/ab.sh "--steps 20 --warmup 5 --no-cpu-baseline" base split > gpurun_out/ab2.log 2>&1
cat gpurun_out/ab.log gpurun_out/ab2.log
