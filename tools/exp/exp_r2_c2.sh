# d=64 ping-pong with one O staging tile per WG (current) vs shared tile (prev); c2 and short-N shapes
FMHA_B200_LIB=build/libfmha_b200_watchdog.so timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -1
S=0,16,17,5,2
for r in 1 2; do
timeout 120 python tools/exp/ab.py cur$r $S
FMHA_B200_LIB=build/var_prev.so timeout 120 python tools/exp/ab.py prev$r $S
done
python tools/prof_phases.py 16 12 512 64
