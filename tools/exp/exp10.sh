timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.txt 2>&1; tail -1 gpurun_out/gpu_tests.txt
for c in c3 c5 c2 c4; do
  timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err
  python -c "import json; j=json.load(open('gpurun_out/b_$c.json')); print('$c', round(j['value'],1), 'e2e', round(j['e2e']['value'],1), j['e2e']['h2d_bytes_per_step'])"
done
