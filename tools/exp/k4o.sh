FMHA_B200_LIB=build/var_k4ow.so timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for rep in 1 2; do
timeout 60 python tools/exp/ab.py base 1,3,4,7,8,9 2>&1 | tail -6
FMHA_B200_LIB=build/var_k4o.so timeout 60 python tools/exp/ab.py k4o 1,3,4,7,8,9 2>&1 | tail -6
done
