# K/V L2 prefetch ahead of the TMA ring (FMHA_KV_PREFETCH) + phase profile
python tools/prof_phases.py
FMHA_B200_LIB=build/prof_pf2.so python tools/prof_phases.py
FMHA_B200_LIB=build/prof_pf4.so python tools/prof_phases.py
S=2,10,11
timeout 120 python tools/exp/ab.py base $S
FMHA_B200_LIB=build/var_pf2.so timeout 120 python tools/exp/ab.py pf2 $S
FMHA_B200_LIB=build/var_pf4.so timeout 120 python tools/exp/ab.py pf4 $S
timeout 120 python tools/exp/ab.py base2 $S
