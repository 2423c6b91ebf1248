export FMHA_TUNE_SPLIT=1
FMHA_B200_LIB=build/var_xsplitw.so timeout 120 python tools/exp/dbs_check.py 2>&1 | tail -15
for rep in 1 2; do
FMHA_TUNE_SPLIT=0 timeout 60 python tools/exp/ab.py base 0,2,6,10,11,18 2>&1 | tail -6
FMHA_B200_LIB=build/var_xsplit.so timeout 60 python tools/exp/ab.py xsplit 0,2,6,10,11,18 2>&1 | tail -6
done
