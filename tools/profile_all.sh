#!/bin/bash
# One-GPU profiling pass: one full ncu capture (with source) per hot kernel on the steady cfg4
# state of tools/kernel_bench.py.  Usage (under gpurun): bash tools/profile_all.sh <tag> [kernels...]
TAG=${1:-r01}; shift
OUT=gpurun_out
KS=${@:-k_integrate:60 k_raycast:1 k_alloc:60 k_sort_blend:1 k_backward:1 k_adam:1 k_chain:1 k_preprocess:1 k_emit:1}
python tools/kernel_bench.py --iters 2 > $OUT/kb_$TAG.log 2>&1 || exit 1
for K in $KS; do
  NAME=${K%%:*}; SKIP=${K##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^${NAME}" -s $SKIP -c 1 \
      -o $OUT/full_${TAG}_${NAME} python tools/kernel_bench.py --iters 2 > $OUT/ncu_${TAG}_${NAME}.log 2>&1
  echo "$NAME ncu exit $?"
done
