#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck on smoke() (cfg1: fuse, raycast,
# render, one refine step through the C ABI).  SURVEY §4 T3.  Logs go to $1 (default gpurun_out/).
out=${1:-gpurun_out}
mkdir -p "$out"
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check no"
  timeout 900 $CS --tool $tool $extra --print-limit 50 \
      python -c "import __graft_entry__ as e; e.smoke()" > "$out/sanitize_$tool.log" 2>&1
  echo "$tool rc=$? $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' "$out/sanitize_$tool.log" | tail -1)"
done
