# c2-like shapes under each d=64 kernel choice (dispatch thresholds forced by env)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{
for rep in 1 2; do
  timeout 300 python tools/exp/ab.py default 0,17,18,12
  FMHA_TUNE_TINY2=100000 timeout 300 python tools/exp/ab.py st64x2 0,17,18,12
  FMHA_TUNE_TINY=100000 timeout 300 python tools/exp/ab.py st128x1 0,17,18,12
  FMHA_TUNE_D64_N=100000 timeout 300 python tools/exp/ab.py pp64 0,17,18,12
done
} > gpurun_out/c2_dispatch.txt 2>&1
