FMHA_B200_LIB=build/libfmha_b200_watchdog.so timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for rep in 1 2; do
FMHA_B200_LIB=build/var_k4.so timeout 200 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-configs 2>/dev/null | python -c "import json,sys; b=json.loads(sys.stdin.read()); print('k4all', b['config']['workload'][:20], round(b['value'],1))"
timeout 200 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-configs 2>/dev/null | python -c "import json,sys; b=json.loads(sys.stdin.read()); print('k4d64', b['config']['workload'][:20], round(b['value'],1))"
FMHA_B200_LIB=build/var_st0.so timeout 200 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-configs 2>/dev/null | python -c "import json,sys; b=json.loads(sys.stdin.read()); print('old', b['config']['workload'][:20], round(b['value'],1))"
done
