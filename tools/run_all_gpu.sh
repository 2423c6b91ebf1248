set -x
timeout 400 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for c in c3 c1 c2 c4 c5; do timeout 300 python bench.py --config $c --steps 50 --warmup 5 $( [ $c != c3 ] && echo --no-cpu-baseline ) > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; python -c "import json; j=json.load(open('gpurun_out/bench_$c.json')); print('$c', round(j['value'],1), 'TF', round(j['ms_per_step'],4), 'ms', 'e2e', j['e2e'] and round(j['e2e']['value'],1), j['clocks'])"; done
