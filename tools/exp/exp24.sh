FMHA_B200_LIB=build/var_spec2.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/gpu_tests_spec2.txt 2>&1; tail -1 gpurun_out/gpu_tests_spec2.txt
for rep in 1 2; do for v in base spec2; do for c in c3 c5 c2; do
  r=$(FMHA_B200_LIB=build/var_$v.so timeout 200 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(round(j['value'],1), j['clocks']['sm_mhz'])")
  echo "$v $c $r"
done; done; done
