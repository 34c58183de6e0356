#!/bin/bash
# One-GPU profiling pass: launch list of the bench command + one full ncu capture per hot kernel.
# Usage (under gpurun): bash tools/profile_all.sh <tag>
TAG=${1:-r01}
OUT=gpurun_out
python tools/kernel_bench.py --iters 2 > $OUT/kb_$TAG.log 2>&1 || exit 1
for K in k_integrate:60 k_raycast:1 k_alloc:60 k_sort_blend:1 k_backward:1 k_adam:1 k_chain:1 k_preprocess:1; do
  NAME=${K%%:*}; SKIP=${K##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^${NAME}" -s $SKIP -c 1 \
      -o $OUT/full_${TAG}_${NAME} python tools/kernel_bench.py --iters 2 > $OUT/ncu_${TAG}_${NAME}.log 2>&1
  echo "$NAME ncu exit $?"
done
