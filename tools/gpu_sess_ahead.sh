timeout 600 python tools/probes/e2e_parts.py 2>&1 | tail -8
bash tools/ab_args.sh "--gpus 1 --steps 20 --warmup 5 --no-cpu-baseline" "ahead12:" "ahead0:--frames-ahead 0" "ahead6:--frames-ahead 6"
