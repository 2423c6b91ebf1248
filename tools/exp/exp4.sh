timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.txt 2>&1; tail -3 gpurun_out/gpu_tests.txt
for c in c3 c5 c2; do timeout 200 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b_$c.json; python -c "import json; j=json.load(open('gpurun_out/b_$c.json')); print('$c', round(j['value'],1), j['clocks'])"; done
FMHA_TUNE_EMU=2 timeout 200 python bench.py --config c3 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e | cut -c1-120
FMHA_TUNE_EMU=0 timeout 200 python bench.py --config c3 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e | cut -c1-120
FMHA_TRACE=1 timeout 120 python tools/trace_timeline.py 4096 128 > gpurun_out/trace_4096_128.txt 2>&1
