# d=64: two-CTA kernel (default) vs ping-pong d=64 (FMHA_TUNE_D64_N=100000) across N, three reps
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{
for rep in 1 2 3; do
  timeout 300 python tools/exp/ab.py d64cta 0,17,18,12,13,1,14
  FMHA_TUNE_D64_N=100000 timeout 300 python tools/exp/ab.py pp64 0,17,18,12,13,1,14
done
} > gpurun_out/c2_dispatch2.txt 2>&1
