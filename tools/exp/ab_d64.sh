for r in 1 2; do
timeout 300 python tools/exp/ab.py base 0,1,12,13,14,15
FMHA_TUNE_D64=2 timeout 300 python tools/exp/ab.py d64e2 0,1,12,13,14,15
FMHA_TUNE_D64=4 timeout 300 python tools/exp/ab.py d64e4 1,13,14
done
