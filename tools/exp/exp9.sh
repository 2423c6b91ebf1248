for v in s44 s40 s42 s20 s00 s22; do for c in c3 c5; do
  r=$(FMHA_KERNEL=split FMHA_B200_LIB=build/var_$v.so timeout 200 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(round(j['value'],1), j['clocks']['sm_mhz'])")
  echo "$v $c $r"
done; done > gpurun_out/exp9.txt 2>&1
for e in 0 2 4; do for c in c3 c5; do
  r=$(FMHA_TUNE_EMU=$e timeout 200 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(round(j['value'],1), j['clocks']['sm_mhz'])")
  echo "base emu$e $c $r"
done; done >> gpurun_out/exp9.txt 2>&1
