for r in 1 2; do
for v in base s21 s20; do
  for c in c3 c4; do
    if [ $v = base ]; then L=""; else L="FMHA_B200_LIB=build/var_$v.so"; fi
    env $L timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/e2e_${v}_$c.json 2>/dev/null
    python -c "
import json; j=json.load(open('gpurun_out/e2e_${v}_$c.json')); e=j['e2e']; print('$v $c', round(e['value'],1), round(e['ms_per_step'],3), 'frac', round(e['roofline']['frac'],3))"
  done
done
done
