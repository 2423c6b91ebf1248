for k in st64 st128; do FMHA_KERNEL=$k timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/gpu_tests_$k.txt 2>&1; echo "$k tests: $(tail -1 gpurun_out/gpu_tests_$k.txt)"; done
for rep in 1 2; do for k in st64 st128 pp; do for c in c3 c5 c2; do
  r=$(FMHA_KERNEL=$k timeout 200 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(round(j['value'],1), j['clocks']['sm_mhz'])")
  echo "$k $c $r"
done; done; done
