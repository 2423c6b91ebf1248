# position-dependent exp2 splits at d=128 through bench.py (variant library built with -DFMHA_EMU_VARIANTS)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export FMHA_B200_LIB=build/var_emuv.so
{
for rep in 1 2; do
  for e in 17 18 19; do
    export FMHA_TUNE_EMU=$e
    for c in c3 c5; do
      timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-configs --no-e2e | python -c "import json,sys; b=json.loads(sys.stdin.readline()); print('emu$e $c', round(b['value'],1), b['clocks']['sm_mhz'], b['clocks']['reasons'])"
    done
  done
done
} > gpurun_out/emu_bench2.txt 2>&1
