set -x
timeout 900 python -m pytest tests/test_gpu_render_refine.py -q -x -k "round" 2>&1 | tail -3
bash tools/ab_args.sh "--gpus 1 --steps 20 --warmup 5" "graph0:" "direct0:--no-graphs" "graph6:GPS_BENCH_HOST_DELAY_US=600" "direct6:GPS_BENCH_HOST_DELAY_US=600 --no-graphs"
