FMHA_KERNEL=si timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_si.txt 2>&1; tail -1 gpurun_out/gpu_tests_si.txt
for k in si pp; do for c in c3 c5 c2; do
  r=$(FMHA_KERNEL=$k timeout 200 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(round(j['value'],1), j['clocks']['sm_mhz'])")
  echo "$k $c $r"
done; done
FMHA_KERNEL=si FMHA_TRACE=1 timeout 120 python tools/trace_timeline.py 4096 128 > gpurun_out/trace_si.txt 2>&1
