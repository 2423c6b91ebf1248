# stall profile of tools/softmax_probe2 V5 (the ping-pong kernel's softmax step in isolation, 1 warp / SMSP)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:ILi5E --launch-skip 1 --launch-count 1 -o gpurun_out/probe5 build/softmax_probe2 > gpurun_out/probe5.log 2>&1
ncu -i gpurun_out/probe5.ncu-rep --page source --csv --print-source sass > gpurun_out/probe5_src.csv
gzip -f gpurun_out/probe5_src.csv; rm -f gpurun_out/probe5.ncu-rep
