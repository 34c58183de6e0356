python -m pytest tests/test_gpu_render_refine.py -m gpu -x -q -k "grad or refine" 2>&1 | tail -2
for rep in 1 2; do
for n in pk80 pk64; do
GPS_LIB=ab/$n/libgps.so python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_${n}_$rep.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/ab_${n}_$rep.json')); print('$n', d['value'], d['kernels']['k_backward']['ms_per_step'])"
done
GPS_BACKWARD_SCALAR=1 GPS_LIB=ab/pk80/libgps.so python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_scalar_$rep.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/ab_scalar_$rep.json')); print('scalar', d['value'], d['kernels']['k_backward']['ms_per_step'])"
done
