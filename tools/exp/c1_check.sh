# c1 (4 Q tiles) kernel choice: one CTA per tile with 128-row K/V steps (default) vs 64-row steps vs ping-pong
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{
for rep in 1 2; do
  for mode in default tiny0 pp; do
    unset FMHA_TUNE_TINY FMHA_TUNE_TINY2
    if [ $mode = tiny0 ]; then export FMHA_TUNE_TINY=0; fi
    if [ $mode = pp ]; then export FMHA_TUNE_TINY=0 FMHA_TUNE_TINY2=0; fi
    timeout 300 python bench.py --config c1 --steps 30 --warmup 5 --no-cpu-baseline --no-configs --no-e2e | python -c "import json,sys; b=json.loads(sys.stdin.readline()); print('$mode c1', round(b['value'],2), round(b['ms_per_step']*1000,2), 'us', b['details']['kernel'][:40] if 'details' in b else '')"
  done
done
} > gpurun_out/c1_check.txt 2>&1
