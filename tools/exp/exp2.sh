FMHA_TRACE=1 timeout 120 python tools/trace_timeline.py 4096 128 > gpurun_out/trace_4096_128.txt 2>&1
FMHA_TRACE=1 timeout 120 python tools/trace_timeline.py 512 64 > gpurun_out/trace_512_64.txt 2>&1
FMHA_TRACE=1 timeout 120 python tools/trace_timeline.py 4096 64 > gpurun_out/trace_4096_64.txt 2>&1
FMHA_TUNE_EMU=0 timeout 200 python bench.py --config c3 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/emu0.json
