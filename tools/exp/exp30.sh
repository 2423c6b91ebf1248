timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.txt 2>&1; tail -1 gpurun_out/gpu_tests.txt
for rep in 1 2; do for bn in 128 64; do
  r=$(FMHA_D256_BN=$bn timeout 200 python bench.py --config c4 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(round(j['value'],1), j['clocks']['sm_mhz'])")
  echo "bn$bn c4 $r"
done; done
FMHA_D256_BN=128 ./paper_2312_11918_b200/fmha-b200 sweep --iterations 20 | tail -1
