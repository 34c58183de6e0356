GPS_LIB=ab/pair75/libgps.so timeout 900 python -m pytest tests/test_gpu_render_refine.py tests/test_gpu_chain.py -q -x 2>&1 | tail -2
GPS_LIB=ab/pair64/libgps.so timeout 900 python -m pytest tests/test_gpu_render_refine.py -q -x -k "gradients" 2>&1 | tail -2
bash tools/ab.sh "--gpus 1 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline" base pair75 pair64
