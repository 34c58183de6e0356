#!/bin/bash
# A/B timing of bench.py argument variants in ONE GPU session (same box, same state):
#   bash tools/ab_args.sh "<common bench args>" "NAME1:ENV=1 --flag" "NAME2:" ...   (under gpurun)
# each spec: NAME:[VAR=value ...] [bench args]
ARGS=$1; shift
for rep in 1 2; do
  for spec in "$@"; do
    n=${spec%%:*}; rest=${spec#*:}
    envs=""; extra=""
    for w in $rest; do
      if [[ $w == *=* && $w != --* ]]; then envs="$envs $w"; else extra="$extra $w"; fi
    done
    env $envs python bench.py $ARGS $extra > gpurun_out/ab_${n}_$rep.json 2> gpurun_out/ab_${n}_$rep.err
    python -c "
import json
d=json.load(open('gpurun_out/ab_${n}_$rep.json'))
k=d['kernels']
print('$n rep$rep', d['value'], (d.get('e2e') or {}).get('value'), d.get('host_enqueue_ms_per_step'), (d.get('e2e') or {}).get('host_enqueue_ms_per_step'), ' '.join(f'{a}={b[\"ms_per_step\"]}' for a,b in k.items() if b['ms_per_step']>0))
" || tail -3 gpurun_out/ab_${n}_$rep.err
  done
done
