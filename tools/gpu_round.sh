#!/bin/bash
# Round-state GPU session (gpurun): GPU tests, smoke, default bench line, ncu launch list.
#   bash tools/gpu_round.sh <tag>
TAG=${1:-r02}
OUT=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/${TAG}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/${TAG}_gputest.log 2>&1; echo "gpu tests exit $?"
tail -3 $OUT/${TAG}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.log 2>&1; echo "smoke exit $?"
timeout 900 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err; echo "bench exit $?"
tail -c 600 $OUT/${TAG}_bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv \
   --log-file $OUT/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline \
   > $OUT/${TAG}_ncu_launch.log 2>&1; echo "ncu launch exit $?"
