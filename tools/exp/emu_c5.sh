# c5 (power-capped) exp2 split: FA4 pattern (default) vs all-MUFU vs 2/16
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{
for rep in 1 2; do
  for e in 17 0 2; do
    export FMHA_TUNE_EMU=$e
    timeout 600 python bench.py --config c5 --steps 20 --warmup 5 --no-cpu-baseline --no-configs --no-e2e | python -c "import json,sys; b=json.loads(sys.stdin.readline()); print('emu$e c5', round(b['value'],1), b['clocks']['sm_mhz'], b['clocks']['reasons'])"
  done
done
} > gpurun_out/emu_c5.txt 2>&1
