timeout 900 python -m pytest tests/test_gpu_render_refine.py tests/test_gpu_chain.py tests/test_gpu_sortfree.py -q -x 2>&1 | tail -2
bash tools/ab.sh "--gpus 1 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline" base new
