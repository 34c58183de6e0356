timeout 900 python tools/probes/e2e_outliers.py 2>&1 | grep -E 'window|upload'
for r in 1 2; do
bash tools/ab_args.sh "--gpus 1 --steps 20 --warmup 5 --no-cpu-baseline" "d$r:" "ng$r:--dense-grid none" "sf$r:--sort-free" "c3$r:--config cfg3"
done
