timeout 120 python tools/exp/ab.py pair 4
FMHA_B200_LIB=build/var_arr1.so timeout 120 python tools/exp/ab.py arr1 4
FMHA_B200_LIB=build/var_arr2.so timeout 120 python tools/exp/ab.py arr2 4
