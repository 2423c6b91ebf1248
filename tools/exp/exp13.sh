ncu --set full --clock-control none -k regex:fmha_fwd -s 3 -c 1 -o gpurun_out/prof_pp python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
FMHA_KERNEL=db ncu --set full --clock-control none -k regex:fmha_fwd -s 3 -c 1 -o gpurun_out/prof_db python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
