S=0,2,10,11,14
FMHA_B200_LIB=build/var_seq0.so python tools/exp/ab.py base $S
python tools/exp/ab.py new $S
FMHA_B200_LIB=build/var_seq0.so python tools/exp/ab.py base2 $S
python tools/exp/ab.py new2 $S
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
