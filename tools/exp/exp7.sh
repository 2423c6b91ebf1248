export FMHA_KERNEL=split
timeout 60 python tools/exp/dbg.py 1 256 1 64 > gpurun_out/dbg1.txt 2>&1
