#!/bin/bash
# scratch GPU session script (gpurun)
for r in 1 2 3 4 5; do
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-profile > gpurun_out/g.json 2> gpurun_out/g.err
  python -c "
import json
d=json.load(open('gpurun_out/g.json'))
print('run $r', d['value'], d['ms_per_step'], d['host_enqueue_ms_per_step'], 'e2e', d['e2e']['value'], d['e2e']['ms_per_step'], d['e2e']['host_enqueue_ms_per_step'], d['e2e']['allocator'])
" || tail -3 gpurun_out/g.err
done
