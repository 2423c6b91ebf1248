set -x
FMHA_TRACE=1 timeout 120 python tools/trace_timeline.py 4096 128 2>&1 | tail -40
for e in 0 4 6 8 12; do FMHA_TUNE_EMU=$e timeout 200 python bench.py --config c3 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('emu $e', round(j['value'],1), j['clocks'])"; done
for e in 0 4 6 8 10 14; do FMHA_TUNE_EMU64=$e timeout 200 python bench.py --config c2 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('c2 emu64 $e', round(j['value'],1))"; done
