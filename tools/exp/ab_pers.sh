FMHA_DEBUG_LAUNCH=1 timeout 300 python tools/exp/ab.py cur 2,3,4,6,7,8,9,10,11
FMHA_TUNE_PAIR128_MIN_N=129 timeout 300 python tools/exp/ab.py pair 2,6,10,11
FMHA_TUNE_PAIR=0 timeout 300 python tools/exp/ab.py nopair 2,3,4,6,7,8,9,10,11
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv
