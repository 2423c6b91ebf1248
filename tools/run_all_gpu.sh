# One gpurun call's worth of checks: GPU tests, every bench config, the CLI
# sweep, and a 1-rank torchrun of the multi-GPU verification path.
set -x
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for c in c3 c1 c2 c4 c5; do timeout 300 python bench.py --config $c --steps 50 --warmup 5 $( [ $c != c3 ] && echo --no-cpu-baseline ) > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; python -c "import json; j=json.load(open('gpurun_out/bench_$c.json')); print('$c', round(j['value'],1), 'TF', round(j['ms_per_step'],4), 'ms', 'e2e', j['e2e'] and round(j['e2e']['value'],1), j['clocks'])"; done
timeout 300 ./paper_2312_11918_b200/fmha-b200 sweep --iterations 20
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 tools/multi_gpu_verify.py --batch 8 --heads 32 --seqlen 4096 --headdim 128 2>&1 | tail -2
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-300
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -1 | cut -c1-600
