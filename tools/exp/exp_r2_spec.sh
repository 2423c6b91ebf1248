# speculative first half (FMHA_SPEC=1, default) vs the row max first (nospec)
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2
S=2,10,11,0,16
timeout 120 python tools/exp/ab.py spec $S
FMHA_B200_LIB=build/var_nospec.so timeout 120 python tools/exp/ab.py nospec $S
timeout 120 python tools/exp/ab.py spec2 $S
FMHA_B200_LIB=build/var_nospec.so timeout 120 python tools/exp/ab.py nospec2 $S
timeout 60 python tools/exp/data_dep.py
