export FMHA_TUNE_DBS=1
FMHA_B200_LIB=build/libfmha_b200_watchdog.so timeout 120 python tools/exp/dbs_check.py 2>&1 | tail -3
FMHA_TUNE_DBS=0 timeout 200 python tools/exp/ab.py base 2,6,7,10,11 2>&1 | tail -5
timeout 200 python tools/exp/ab.py dbs 2,6,7,10,11 2>&1 | tail -5
for v in ss32 ss100 noidle; do FMHA_B200_LIB=build/var_$v.so timeout 200 python tools/exp/ab.py $v 2,6,7,10,11 2>&1 | tail -5; done
