# exp2 split of the d=128 ping-pong kernel after the padded-step split (FMHA_TUNE_EMU selects the instantiation)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{
for rep in 1 2; do
  for e in 4 2 6 17 0; do FMHA_TUNE_EMU=$e timeout 300 python tools/exp/ab.py emu$e 2,6,11; done
done
} > gpurun_out/emu_retune.txt 2>&1
