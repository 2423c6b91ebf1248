# A/B of two library builds: ab_var.sh BASE_SO VAR_SO SHAPES [pytest -k expr run on VAR]
# ("-" = the in-tree paper_2312_11918_b200/libfmha_b200.so)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B=$1; V=$2; SH=$3
lib() { if [ "$1" = "-" ]; then echo paper_2312_11918_b200/libfmha_b200.so; else echo $1; fi; }
{
for rep in 1 2; do
  FMHA_B200_LIB=$(lib $B) timeout 300 python tools/exp/ab.py base $SH
  FMHA_B200_LIB=$(lib $V) timeout 300 python tools/exp/ab.py var $SH
done
if [ -n "$4" ]; then FMHA_B200_LIB=$(lib $V) timeout 900 python -m pytest tests -m gpu -x -q -k "$4" 2>&1 | tail -3; fi
} > gpurun_out/ab_var.txt 2>&1
