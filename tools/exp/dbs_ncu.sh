mkdir -p gpurun_out
FMHA_TUNE_DBS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:fmha_fwd -s 3 -c 1 -o gpurun_out/prof_dbs_c3 python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-configs > /dev/null 2>&1
ls -la gpurun_out
