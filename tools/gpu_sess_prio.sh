bash tools/ab_args.sh "--gpus 1 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e" "base:" "view1:--view-priority -1" "view2:--view-priority -2"
