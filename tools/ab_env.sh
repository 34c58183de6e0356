#!/bin/bash
# A/B timing of environment-selected variants in ONE GPU session (same box, same state):
#   bash tools/ab_env.sh "<bench args>" "NAME1:VAR=1" "NAME2:" ...   (under gpurun)
ARGS=$1; shift
for rep in 1 2; do
  for spec in "$@"; do
    n=${spec%%:*}; envs=${spec#*:}
    env $envs python bench.py $ARGS > gpurun_out/ab_${n}_$rep.json 2> gpurun_out/ab_${n}_$rep.err
    python -c "
import json,sys
d=json.load(open('gpurun_out/ab_${n}_$rep.json'))
k=d['kernels']
print('$n rep$rep', d['value'], (d.get('e2e') or {}).get('value'), ' '.join(f'{a}={b[\"ms_per_step\"]}' for a,b in k.items() if b['ms_per_step']>0))
" || tail -3 gpurun_out/ab_${n}_$rep.err
  done
done
