timeout 900 python -m pytest tests/test_gpu_render_refine.py tests/test_gpu_pipeline.py tests/test_gpu_checked.py -q -x 2>&1 | tail -2
for r in 1 2; do
bash tools/ab.sh "--gpus 1 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline" base new
done
