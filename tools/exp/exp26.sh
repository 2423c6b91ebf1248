FMHA_B200_LIB=build/var_trace_noexp.so FMHA_TRACE=1 timeout 120 python tools/trace_timeline.py 4096 128 > gpurun_out/trace_noexp.txt 2>&1
FMHA_B200_LIB=build/var_trace_base.so FMHA_TRACE=1 timeout 120 python tools/trace_timeline.py 4096 128 > gpurun_out/trace_base.txt 2>&1
