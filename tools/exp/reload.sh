FMHA_B200_LIB=build/var_reload.so timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "not double_buffered" 2>&1 | tail -2
for rep in 1 2; do
timeout 60 python tools/exp/ab.py base 0,2,3,6,10,11 2>&1 | tail -6
FMHA_B200_LIB=build/var_reload.so timeout 60 python tools/exp/ab.py reload 0,2,3,6,10,11 2>&1 | tail -6
done
FMHA_B200_LIB=build/libfmha_b200_profreload.so python tools/prof_phases.py 2>&1 | tail -4
