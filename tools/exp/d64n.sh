for rep in 1 2; do
for n in 1024 256; do
for c in c2; do FMHA_TUNE_D64_N=$n timeout 200 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-configs 2>/dev/null | python -c "import json,sys; b=json.loads(sys.stdin.read()); print('d64_n=$n', b['config']['workload'][:12], round(b['value'],1), b['details']['kernel'][:40])"; done
FMHA_TUNE_D64_N=$n timeout 60 python tools/exp/ab.py n$n 0,16,17,18 2>&1 | tail -4
done
done
