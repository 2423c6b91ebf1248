FMHA_B200_LIB=build/var_k4w.so timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_boundaries.py -m gpu -q -x -k "not opt_in" 2>&1 | tail -1
for rep in 1 2 3; do
timeout 60 python tools/exp/ab.py base 0,2,3,6,10,11,18 2>&1 | tail -7
FMHA_B200_LIB=build/var_k4.so timeout 60 python tools/exp/ab.py k4 0,2,3,6,10,11,18 2>&1 | tail -7
done
