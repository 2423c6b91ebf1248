for r in 1 2 3; do
timeout 300 python tools/exp/ab.py half 4,3
FMHA_B200_LIB=build/var_head.so timeout 300 python tools/exp/ab.py head 4,3
done
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
