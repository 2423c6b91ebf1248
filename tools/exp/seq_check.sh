# FMHA_SEQ (exponential phases of the two softmax WGs in strict turns): phase profile + A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{
echo "== phases default"; FMHA_B200_LIB=build/libfmha_b200_prof.so timeout 300 python tools/prof_phases.py
echo "== phases FMHA_SEQ=1"; FMHA_B200_LIB=build/libfmha_b200_profseq.so timeout 300 python tools/prof_phases.py
for rep in 1 2; do
  timeout 300 python tools/exp/ab.py base 2,6,11
  FMHA_B200_LIB=build/libfmha_b200_seq.so timeout 300 python tools/exp/ab.py seq 2,6,11
done
} > gpurun_out/seq_check.txt 2>&1
