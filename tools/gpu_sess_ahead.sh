for r in 1 2; do
bash tools/ab_args.sh "--gpus 1 --steps 20 --warmup 5 --no-cpu-baseline" "d0$r:" "d20$r:--frames-ahead 20" "ng0$r:--dense-grid none" "ng20$r:--dense-grid none --frames-ahead 20"
done
