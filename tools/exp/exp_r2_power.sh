# burst (ab.py) and sustained (2 s back to back, power-capped) throughput of the d=128 kernels on c3
S=2
timeout 120 python tools/exp/ab.py pp $S
FMHA_TUNE_PAIR128_N=1024 timeout 120 python tools/exp/ab.py pair $S
FMHA_TUNE_EMU=0 timeout 120 python tools/exp/ab.py pp_emu0 $S
FMHA_TUNE_EMU=8 timeout 120 python tools/exp/ab.py pp_emu8 $S
python tools/exp/clock_under_load.py c3
FMHA_TUNE_PAIR128_N=1024 python tools/exp/clock_under_load.py c3
FMHA_TUNE_EMU=0 python tools/exp/clock_under_load.py c3
FMHA_TUNE_EMU=8 python tools/exp/clock_under_load.py c3
FMHA_TUNE_PAIR128_N=1000000 python tools/exp/clock_under_load.py c5
python tools/exp/clock_under_load.py c5
