timeout 600 python -m pytest tests -m gpu -q -x -k "host" > gpurun_out/gpu_tests_host.txt 2>&1; tail -3 gpurun_out/gpu_tests_host.txt
