timeout 300 python tools/exp/ab.py base 2,3,6,7,8,9,10,11
FMHA_B200_LIB=build/var_e2.so FMHA_TUNE_PAIR128=64 timeout 300 python tools/exp/ab.py p64e2 2,3,6,7,8,9,10,11
timeout 300 python tools/exp/ab.py base 2,3,6,7,8,9,10,11
FMHA_B200_LIB=build/var_e2.so FMHA_TUNE_PAIR128=64 timeout 300 python tools/exp/ab.py p64e2 2,3,6,7,8,9,10,11
