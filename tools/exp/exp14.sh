FMHA_TRACE=1 timeout 120 python tools/trace_timeline.py 4096 128 > gpurun_out/trace_pp.txt 2>&1
