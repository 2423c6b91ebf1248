FMHA_KERNEL=db timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_db.txt 2>&1; tail -1 gpurun_out/gpu_tests_db.txt
for k in db pingpong; do for c in c3 c2 c5; do
  r=$(FMHA_KERNEL=$k timeout 200 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(round(j['value'],1), j['clocks']['sm_mhz'])")
  echo "$k $c $r"
done; done
