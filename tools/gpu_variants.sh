#!/bin/bash
# Bench lines for the other north_star streams and windows (gpurun): cfg2 (TUM-shaped), cfg3
# (Replica-shaped), cfg4 late window (frames 2500+), cfg4 without the dense block grid.
TAG=${1:-r02}
O=gpurun_out
timeout 900 python bench.py --config cfg2 --no-cpu-baseline > $O/${TAG}_bench_cfg2.json 2> $O/${TAG}_bench_cfg2.err; echo "cfg2 $?"
timeout 900 python bench.py --config cfg3 --no-cpu-baseline > $O/${TAG}_bench_cfg3.json 2> $O/${TAG}_bench_cfg3.err; echo "cfg3 $?"
timeout 900 python bench.py --dense-grid none --no-cpu-baseline > $O/${TAG}_bench_nogrid.json 2> $O/${TAG}_bench_nogrid.err; echo "nogrid $?"
timeout 1500 python bench.py --history 2500 --no-cpu-baseline > $O/${TAG}_bench_late.json 2> $O/${TAG}_bench_late.err; echo "late $?"
for f in cfg2 cfg3 nogrid late; do python -c "
import json; d=json.load(open('$O/${TAG}_bench_$f.json')); print('$f', d['value'], (d.get('e2e') or {}).get('value'), d['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'])" 2>/dev/null || tail -2 $O/${TAG}_bench_$f.err; done
