FMHA_KERNEL=sts timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/gpu_tests_sts.txt 2>&1; echo "sts tests: $(tail -1 gpurun_out/gpu_tests_sts.txt)"
for rep in 1 2; do for k in sts pp; do for c in c3 c5 c2; do
  r=$(FMHA_KERNEL=$k timeout 200 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(round(j['value'],1), j['clocks']['sm_mhz'])")
  echo "$k $c $r"
done; done; done
FMHA_KERNEL=sts ./paper_2312_11918_b200/fmha-b200 sweep --iterations 20 | head -2
