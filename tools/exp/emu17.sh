FMHA_TUNE_EMU=17 timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "large or ragged or small" 2>&1 | tail -1
for rep in 1 2 3; do
FMHA_TUNE_EMU=4 timeout 60 python tools/exp/ab.py e4 2,6,10,11 2>&1 | tail -4
FMHA_TUNE_EMU=17 timeout 60 python tools/exp/ab.py e17 2,6,10,11 2>&1 | tail -4
done
