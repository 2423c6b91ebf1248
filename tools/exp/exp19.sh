ncu --set full --clock-control none -s 3 -c 1 -k regex:'^(?!.*(elementwise|distribution|copy|fill)).*' -o gpurun_out/prof_cudnn python tools/exp/calib_ncu.py > gpurun_out/ncu_cudnn.log 2>&1
tail -5 gpurun_out/ncu_cudnn.log
