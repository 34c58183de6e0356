GPS_LIB=ab/bl6/libgps.so timeout 900 python -m pytest tests/test_gpu_render_refine.py -q -x -k "cfg1 or two_pixel" 2>&1 | tail -1
for r in 1 2; do
bash tools/ab.sh "--gpus 1 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline" base bl6 bl7
done
