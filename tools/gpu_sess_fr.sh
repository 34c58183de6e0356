for r in 1 2; do
bash tools/ab_args.sh "--gpus 1 --steps 20 --warmup 5 --no-cpu-baseline" "both$r:" "roundonly$r:--no-frame-graphs" "none$r:--no-graphs"
done
