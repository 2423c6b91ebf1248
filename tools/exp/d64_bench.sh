# d=64 dispatch check through bench.py (c2, L2 flushed) and the CLI Table-1 sweep, default vs ping-pong d=64
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{
for rep in 1 2; do
  for mode in default pp64; do
    if [ $mode = pp64 ]; then export FMHA_TUNE_D64_N=100000; else unset FMHA_TUNE_D64_N; fi
    echo "== $mode rep $rep"
    timeout 300 python bench.py --config c2 --steps 30 --warmup 5 --no-cpu-baseline --no-configs | python -c "import json,sys; b=json.loads(sys.stdin.readline()); print('c2', round(b['value'],1), b['clocks'], b['e2e']['value'] if isinstance(b.get('e2e'),dict) else '')"
    timeout 300 ./paper_2312_11918_b200/fmha-b200 sweep --iterations 20 2>&1 | grep "d=64"
  done
done
} > gpurun_out/d64_bench.txt 2>&1
