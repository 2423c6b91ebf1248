for rep in 1 2; do for v in cluster spread; do for c in c3 c5 c4 c2; do
  r=$(FMHA_B200_LIB=build/var_$v.so timeout 200 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(round(j['value'],1), j['clocks']['sm_mhz'])")
  echo "$v $c $r"
done; done; done
for e in 4 6; do r=$(FMHA_TUNE_EMU=$e FMHA_B200_LIB=build/var_spread.so timeout 200 python bench.py --config c3 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(round(j['value'],1))"); echo "spread emu$e c3 $r"; done
