for rep in 1 2; do for v in pf0 pf4 pf8 pf32; do for c in c2 c3 c1; do
  r=$(FMHA_B200_LIB=build/var_$v.so timeout 200 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(round(j['value'],1), j['clocks']['sm_mhz'])")
  echo "$v $c $r"
done; done; done
