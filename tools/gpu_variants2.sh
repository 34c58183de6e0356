#!/bin/bash
# NEXT-row bench variants on the current kernels (gpurun): sort-free renderer (+ warp backward),
# ICP tracking, Gaussian adding/removal, all views per iteration, ScanNet++-sized frames
TAG=${1:-r02h}
O=gpurun_out
run() { name=$1; shift; timeout 900 python bench.py --no-cpu-baseline "$@" > $O/${TAG}_bench_$name.json 2> $O/${TAG}_bench_$name.err; echo "$name $?"; }
run sortfree --sort-free
run sortfree_warpbwd --sort-free --backward 1
run track --track
run manage --manage-gaussians
run allviews --all-views
run scannetpp --config scannetpp
for f in sortfree sortfree_warpbwd track manage allviews scannetpp; do python -c "
import json; d=json.load(open('$O/${TAG}_bench_$f.json')); print('$f', d['value'], (d.get('e2e') or {}).get('value'), d['ms_per_step'], (d.get('tracking') or {}).get('ate_rmse_mm'))" 2>/dev/null || tail -2 $O/${TAG}_bench_$f.err; done
