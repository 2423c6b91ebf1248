for rep in 1 2; do
timeout 60 python tools/exp/ab.py r192 0,2,6,10,11 2>&1 | tail -5
for v in r200 r208; do FMHA_B200_LIB=build/var_$v.so timeout 60 python tools/exp/ab.py $v 0,2,6,10,11 2>&1 | tail -5; done
done
