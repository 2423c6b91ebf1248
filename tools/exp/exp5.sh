for v in base c4 c4d c4ds spec spin c4spin; do
  for c in c3 c2; do
    r=$(FMHA_B200_LIB=build/var_$v.so timeout 200 python bench.py --config $c --steps 40 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(round(j['value'],1))")
    echo "$v $c $r"
  done
done > gpurun_out/exp5.txt 2>&1
