python tools/exp/ab.py base
FMHA_TUNE_ST=64 python tools/exp/ab.py st64 0,1,2,5
python tools/exp/ab.py base 0,1,2
FMHA_TUNE_ST=64 python tools/exp/ab.py st64 0,1,2
