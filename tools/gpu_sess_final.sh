TAG=$1
bash tools/gpu_round.sh $TAG
timeout 900 python bench.py --steps 10 --warmup 5 --no-e2e --no-cpu-baseline --timeline gpurun_out/${TAG}_timeline.json > gpurun_out/${TAG}_tl.json 2> gpurun_out/${TAG}_tl.err; echo "timeline exit $?"
