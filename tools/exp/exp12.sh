timeout 120 python tools/trace_db.py 4096 128 > gpurun_out/trace_db.txt 2>&1
