# O staged in the Q buffer + 5-slot K/V ring (FMHA_O_IN_Q=1, default) vs 4 slots + separate staging
FMHA_B200_LIB=build/libfmha_b200_watchdog.so timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_boundaries.py -m gpu -q -x 2>&1 | tail -2
python tools/prof_phases.py
S=2,10,11,0
timeout 120 python tools/exp/ab.py oinq $S
FMHA_B200_LIB=build/var_oinq0.so timeout 120 python tools/exp/ab.py oinq0 $S
timeout 120 python tools/exp/ab.py oinq_2 $S
FMHA_B200_LIB=build/var_oinq0.so timeout 120 python tools/exp/ab.py oinq0_2 $S
