bash tools/ab_args.sh "--gpus 1 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e" "rhigh:" "fhigh:--refine-priority 0 --fusion-priority -1" "equal:--refine-priority 0"
