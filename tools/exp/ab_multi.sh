# interleaved A/B of several library builds: ab_multi.sh SHAPES LIB1 LIB2 ... ("-" = in-tree build)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SH=$1; shift
{
for rep in 1 2; do
  for L in "$@"; do
    if [ "$L" = "-" ]; then LL=paper_2312_11918_b200/libfmha_b200.so; T=base; else LL=$L; T=$(basename $L .so); fi
    FMHA_B200_LIB=$LL timeout 300 python tools/exp/ab.py $T $SH
  done
done
} > gpurun_out/ab_multi.txt 2>&1
