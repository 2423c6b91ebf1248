mkdir -p gpurun_out
export FMHA_TUNE_DBS=1
FMHA_B200_LIB=build/libfmha_b200_watchdog.so timeout 120 python tools/exp/dbs_check.py 2>&1 | tail -20
echo "--- timing"
FMHA_TUNE_DBS=0 timeout 200 python tools/exp/ab.py base 2,6,7,10,11 2>&1 | tail -5
FMHA_TUNE_DBS=1 timeout 200 python tools/exp/ab.py dbs 2,6,7,10,11 2>&1 | tail -5
FMHA_TUNE_DBS=1 FMHA_TUNE_EMU=6 timeout 200 python tools/exp/ab.py dbs6 2,6,7,10,11 2>&1 | tail -5
FMHA_TUNE_DBS=1 FMHA_TUNE_EMU=8 timeout 200 python tools/exp/ab.py dbs8 2,6,7,10,11 2>&1 | tail -5
