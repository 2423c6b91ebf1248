for rep in 1 2; do for e in 4 6 8; do for c in c3 c5; do
  r=$(FMHA_TUNE_EMU=$e timeout 200 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(round(j['value'],1), j['clocks']['sm_mhz'])")
  echo "emu$e $c $r"
done; done;
for e in 4 6 8; do
  r=$(FMHA_TUNE_EMU64=$e timeout 200 python bench.py --config c2 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(round(j['value'],1))")
  echo "emu64_$e c2 $r"
done; done
