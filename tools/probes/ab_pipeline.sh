# A/B of two pipeline.py versions on one box (scratch)
P=paper_2509_11574_b200/pipeline.py
for rep in 1 2; do
for v in old new; do
cp tools/probes/pipeline_$v.py $P
GPS_BENCH_HOST_DELAY_US=1000 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab_pl_${v}_$rep.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/ab_pl_${v}_$rep.json')); print('$v', d['value'], d['e2e']['value'], d['e2e']['host_enqueue_ms_per_step'])"
done; done
cp tools/probes/pipeline_new.py $P
