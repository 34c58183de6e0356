python -m pytest tests/test_gpu_fuse_raycast.py tests/test_gpu_edges.py tests/test_gpu_chain.py tests/test_gpu_pipeline.py tests/test_gpu_checked.py -m gpu -x -q 2>&1 | tail -3
for rep in 1 2; do
for n in r107 r80 r64; do
GPS_LIB=ab/$n/libgps.so python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_${n}_$rep.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/ab_${n}_$rep.json')); print('$n', d['value'], d['kernels']['k_integrate']['ms_per_step'])"
done
GPS_INTEGRATE_PAIRS=1 GPS_LIB=ab/r80/libgps.so python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_pairs_$rep.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/ab_pairs_$rep.json')); print('pairs', d['value'], d['kernels']['k_integrate']['ms_per_step'])"
done
