FMHA_B200_LIB=build/var_fusedw.so timeout 900 python -m pytest tests -m gpu -q -x -k "not sanitizer and not dropin" 2>&1 | tail -1
for rep in 1 2 3; do
timeout 60 python tools/exp/ab.py base 0,1,14,15,18 2>&1 | tail -5
FMHA_B200_LIB=build/var_fused.so timeout 60 python tools/exp/ab.py fused 0,1,14,15,18 2>&1 | tail -5
done
