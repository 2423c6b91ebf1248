for rep in 1 2; do
FMHA_B200_LIB=build/var_st0.so timeout 200 python tools/exp/ab.py st0 0,2,6,7,10,11 2>&1 | tail -6
timeout 200 python tools/exp/ab.py st256 0,2,6,7,10,11 2>&1 | tail -6
for v in ss32 ss64 ss128; do FMHA_B200_LIB=build/var_$v.so timeout 200 python tools/exp/ab.py $v 0,2,6,7,10,11 2>&1 | tail -6; done
done
