FMHA_TRACE=1 timeout 120 python tools/trace_timeline.py 4096 128 > gpurun_out/trace_4096_128.txt 2>&1
FMHA_TRACE=1 timeout 120 python tools/trace_timeline.py 4096 64 > gpurun_out/trace_4096_64.txt 2>&1
