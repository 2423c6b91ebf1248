for r in 1 2; do
timeout 300 python tools/exp/ab.py base 0,5,16,17,18
FMHA_TUNE_D64S=1 timeout 300 python tools/exp/ab.py d64s 0,5,16,17,18
FMHA_TUNE_D64S=2 timeout 300 python tools/exp/ab.py d64se2 0,17
done
FMHA_TUNE_D64S=1 timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
