# the other north_star streams and the NEXT-row variants on the final kernels (one box)
T=r02m
run() { n=$1; shift; timeout 1200 python bench.py --no-cpu-baseline "$@" > gpurun_out/${T}_bench_$n.json 2> gpurun_out/${T}_bench_$n.err; python -c "
import json; d=json.load(open('gpurun_out/${T}_bench_$n.json')); print('$n', d['value'], (d.get('e2e') or {}).get('value'))" || tail -2 gpurun_out/${T}_bench_$n.err; }
run default
run cfg2 --config cfg2
run cfg3 --config cfg3
run nogrid --dense-grid none
run sortfree --sort-free
run track --track
run manage --manage-gaussians
run allviews --all-views
run scannetpp --config scannetpp
run late --history 2560
