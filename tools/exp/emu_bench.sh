# exp2 split of the d=128 ping-pong kernel through bench.py (c3 with L2 flush, c5 power-capped)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{
for rep in 1 2; do
  for e in 4 17 2; do
    export FMHA_TUNE_EMU=$e
    for c in c3 c5; do
      timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-configs --no-e2e | python -c "import json,sys; b=json.loads(sys.stdin.readline()); print('emu$e $c', round(b['value'],1), b['clocks']['sm_mhz'], b['clocks']['reasons'])"
    done
  done
done
} > gpurun_out/emu_bench.txt 2>&1
