# split-row kernel: correctness under the watchdog build, then A/B
export FMHA_TUNE_SPLIT=1
FMHA_B200_LIB=build/libfmha_b200_watchdog.so timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "d128 or c3 or small_full or ragged or strided or custom or kv_perm or host or identical or single" 2>&1 | tail -3
S=2,10,11,0
FMHA_TUNE_SPLIT=0 timeout 120 python tools/exp/ab.py base $S
FMHA_TUNE_SPLIT=1 timeout 120 python tools/exp/ab.py split4 $S
FMHA_TUNE_SPLIT=1 FMHA_TUNE_EMU=6 timeout 120 python tools/exp/ab.py split6 $S
FMHA_TUNE_SPLIT=1 FMHA_TUNE_EMU=2 timeout 120 python tools/exp/ab.py split2 $S
FMHA_TUNE_SPLIT=0 timeout 120 python tools/exp/ab.py base2 $S
