# c5 through bench.py and d=128 N=8192 bf16, CTA pairs (default) vs ping-pong (FMHA_TUNE_PAIR128_N=1000000)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{
for rep in 1 2; do
  for mode in pair pp; do
    if [ $mode = pp ]; then export FMHA_TUNE_PAIR128_N=1000000; else unset FMHA_TUNE_PAIR128_N; fi
    timeout 600 python bench.py --config c5 --steps 20 --warmup 5 --no-cpu-baseline --no-configs --no-e2e | python -c "import json,sys; b=json.loads(sys.stdin.readline()); print('$mode c5', round(b['value'],1), b['clocks'])"
    timeout 300 python tools/exp/ab.py $mode 8,7
  done
done
} > gpurun_out/pair_vs_pp2.txt 2>&1
