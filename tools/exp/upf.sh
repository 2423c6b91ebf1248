for rep in 1 2; do
for v in upf0 upf64; do FMHA_B200_LIB=build/var_$v.so timeout 120 python tools/exp/flush_mode.py 2>&1 | grep "memset " | sed "s/^/$v /"; done
timeout 120 python tools/exp/flush_mode.py 2>&1 | grep "memset " | sed "s/^/upf8 /"
done
