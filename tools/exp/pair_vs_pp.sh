# d=128 long sequences: CTA-pair kernel (default, N >= 8192) vs the ping-pong kernel (FMHA_TUNE_PAIR128_N=100000)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{
for rep in 1 2; do
  timeout 600 python tools/exp/ab.py pair 7,8,9,3
  FMHA_TUNE_PAIR128_N=1000000 timeout 600 python tools/exp/ab.py pp 7,8,9,3
done
} > gpurun_out/pair_vs_pp.txt 2>&1
