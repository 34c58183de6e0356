bash tools/ab_args.sh "--gpus 1 --steps 20 --warmup 5 --no-cpu-baseline" "d0:" "d300:GPS_BENCH_HOST_DELAY_US=300" "d600:GPS_BENCH_HOST_DELAY_US=600" "d900:GPS_BENCH_HOST_DELAY_US=900"
