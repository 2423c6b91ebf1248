for c in c2 c1 c3; do timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/e2e_$c.json 2>/dev/null; python -c "
import json; j=json.load(open('gpurun_out/e2e_$c.json')); e=j['e2e']; print('$c', round(j['value'],1), 'e2e', round(e['value'],2), round(e['ms_per_step'],3), 'ms', 'frac', round(e['roofline']['frac'],3))"; done
timeout 600 python -m pytest tests -m gpu -q -x -k "host" 2>&1 | tail -2
