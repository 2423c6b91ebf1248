timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_all.txt 2>&1; tail -2 gpurun_out/gpu_tests_all.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
for c in c3 c1 c2 c4 c5; do timeout 300 python bench.py --config $c --steps 50 --warmup 5 $( [ $c != c3 ] && echo --no-cpu-baseline ) > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; python -c "import json; j=json.load(open('gpurun_out/bench_$c.json')); print('$c', round(j['value'],1), 'TF', round(j['ms_per_step'],4), 'ms', 'e2e', j['e2e'] and round(j['e2e']['value'],1), j['clocks'])"; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>/dev/null; cut -c1-300 gpurun_out/bench_ref.json
