# TMA-store epilogues in the pair / single-CTA / d=64 two-CTA kernels (current) vs row-per-thread st.global (prev)
FMHA_B200_LIB=build/libfmha_b200_watchdog.so timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
S=4,3,1,14,8,16,17
timeout 200 python tools/exp/ab.py cur $S
FMHA_B200_LIB=build/var_prev.so timeout 200 python tools/exp/ab.py prev $S
timeout 200 python tools/exp/ab.py cur2 $S
FMHA_B200_LIB=build/var_prev.so timeout 200 python tools/exp/ab.py prev2 $S
