FMHA_B200_LIB=build/libfmha_b200_watchdog.so timeout 600 python -m pytest tests -m gpu -q -x -k "d64 or config1 or config2 or small or ragged or strided or single_key or identical or custom_scale or launch_count or permutation or linearity or boundaries" 2>&1 | tail -2
for rep in 1 2 3; do
FMHA_B200_LIB=build/var_noepi.so timeout 200 python tools/exp/ab.py noepi 0,10,16,17,18 2>&1 | tail -5
timeout 200 python tools/exp/ab.py epiwg 0,10,16,17,18 2>&1 | tail -5
done
