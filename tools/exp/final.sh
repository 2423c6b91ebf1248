timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_all.txt 2>&1; tail -2 gpurun_out/gpu_tests_all.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
for c in c3 c1 c2 c4 c5; do timeout 300 python bench.py --config $c --steps 50 --warmup 5 $( [ $c != c3 ] && echo --no-cpu-baseline ) > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; python -c "import json; j=json.load(open('gpurun_out/bench_$c.json')); print('$c', round(j['value'],1), 'TF', round(j['ms_per_step'],4), 'ms', 'e2e', j['e2e'] and round(j['e2e']['value'],1), j['clocks'])"; done
timeout 300 ./paper_2312_11918_b200/fmha-b200 sweep --iterations 20 > gpurun_out/sweep.txt 2>&1; cat gpurun_out/sweep.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:fmha_fwd -s 3 -c 1 -o gpurun_out/prof_c3 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none -k regex:fmha_fwd -s 3 -c 1 -o gpurun_out/prof_c4 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_torchrun.json 2>/dev/null; cut -c1-200 gpurun_out/bench_torchrun.json
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>/dev/null; cut -c1-200 gpurun_out/bench_ref.json
ncu --set full --clock-control none -k regex:fmha_fwd -s 3 -c 1 -o gpurun_out/prof_c5 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
