for r in 1 2 3; do timeout 900 python bench.py > gpurun_out/rep_$r.json 2> gpurun_out/rep_$r.err; python -c "
import json; d=json.load(open('gpurun_out/rep_$r.json')); print('rep$r', d['value'], d['e2e']['value'], d['clocks']['sm_mhz'], d['cpu_baseline']['value'] if d.get('cpu_baseline') else None)"; done
