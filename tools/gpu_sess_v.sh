for r in 1 2; do
bash tools/ab.sh "--gpus 1 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline" base ig4 ig12 ig16
done
