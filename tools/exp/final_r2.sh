# Round-2 measurement run (one gpurun call): GPU suite, smoke, bench (default line with every config),
# reference arm, CLI sweep, ncu launch list + full captures, sustained (power-capped) throughput.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_all.txt 2>&1; tail -2 gpurun_out/gpu_tests_all.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -3 gpurun_out/smoke.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; cut -c1-300 gpurun_out/bench_default.json
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cut -c1-300 gpurun_out/bench_ref.json
timeout 300 ./paper_2312_11918_b200/fmha-b200 sweep --iterations 20 > gpurun_out/sweep.txt 2>&1; tail -12 gpurun_out/sweep.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-configs > /dev/null 2>&1
for c in c3 c2 c4 c5; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:fmha_fwd -s 3 -c 1 -o gpurun_out/prof_$c python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-configs > /dev/null 2>&1
  # the pull back is capped at 64 MiB: keep c3's report, export the others' raw metrics
  if [ $c = c3 ]; then ncu -i gpurun_out/prof_c3.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/prof_c3_source.csv.gz; fi
  if [ $c != c3 ]; then ncu -i gpurun_out/prof_$c.ncu-rep --page raw --csv > gpurun_out/prof_${c}_raw.csv 2>/dev/null && rm -f gpurun_out/prof_$c.ncu-rep; fi
done
python tools/exp/clock_under_load.py c3 c5 c4 c2 > gpurun_out/sustained.txt 2>&1; cat gpurun_out/sustained.txt
make -s prof > /dev/null 2>&1; python tools/prof_phases.py > gpurun_out/phases_c3.txt 2>&1; python tools/prof_phases.py 16 12 512 64 > gpurun_out/phases_c2.txt 2>&1; cat gpurun_out/phases_c3.txt
ls -la gpurun_out
bash tools/exp/epi_probe.sh > gpurun_out/epilogue_probe.txt 2>&1; cat gpurun_out/epilogue_probe.txt
