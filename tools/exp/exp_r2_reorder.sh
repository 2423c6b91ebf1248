# K(j) waited after PV0(j-1) issue + early V release (current) vs HEAD
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -1
python tools/prof_phases.py
S=2,10,11,0
timeout 120 python tools/exp/ab.py cur $S
FMHA_B200_LIB=build/var_prev.so timeout 120 python tools/exp/ab.py prev $S
timeout 120 python tools/exp/ab.py cur2 $S
FMHA_B200_LIB=build/var_prev.so timeout 120 python tools/exp/ab.py prev2 $S
