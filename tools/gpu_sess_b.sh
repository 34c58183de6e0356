bash tools/ab_env.sh "--steps 20 --warmup 5 --no-cpu-baseline --no-e2e" "base:" "norange:GPS_NO_RANGE=1" > gpurun_out/ab_range.log 2>&1
cat gpurun_out/ab_range.log
bash tools/profile_all.sh r02b k_integrate:60 k_raycast:1 k_backward:1 k_sort_blend:1 k_chain_adam:1 k_preprocess:1
