#!/bin/bash
# A/B timing of library variants in ONE GPU session (same box, same state): for each built
# variant ab/<name>/libgps.so (python paper_2509_11574_b200/build.py --out ab/<name>/libgps.so),
# run the same bench command with GPS_LIB pointing at it, twice, interleaved.
#   bash tools/ab.sh "<bench args>" name1 name2 ...      (under gpurun)
ARGS=$1; shift
for rep in 1 2; do
  for n in "$@"; do
    GPS_LIB=ab/$n/libgps.so python bench.py $ARGS > gpurun_out/ab_${n}_$rep.json 2> gpurun_out/ab_${n}_$rep.err
    python -c "
import json,sys
d=json.load(open('gpurun_out/ab_${n}_$rep.json'))
k=d['kernels']
print('$n rep$rep', d['value'], (d.get('e2e') or {}).get('value'), ' '.join(f'{a}={b[\"ms_per_step\"]}' for a,b in k.items() if b['ms_per_step']>0))
" || tail -3 gpurun_out/ab_${n}_$rep.err
  done
done
