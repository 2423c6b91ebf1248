# source-level stall profile of the two-CTA d=64 kernel on the Table-1 d=64 shape (L=4, h=32, N=4096)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fmha_fwd_d64 -c 1 -o gpurun_out/d64src python tools/exp/ab.py base 1 > gpurun_out/d64src.log 2>&1
ncu -i gpurun_out/d64src.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/d64_source.csv.gz
ncu -i gpurun_out/d64src.ncu-rep --page raw --csv > gpurun_out/d64_raw.csv 2>/dev/null
rm -f gpurun_out/d64src.ncu-rep
