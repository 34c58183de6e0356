bash tools/ab_args.sh "--gpus 1 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e" "off:" "p38:GPS_L2_PERSIST_MB=38" "m38:GPS_L2_PERSIST_MB=38 GPS_L2_PERSIST_WHAT=m" "p76:GPS_L2_PERSIST_MB=76"
