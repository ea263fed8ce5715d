timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -3
timeout 300 python tools/probe_scaling.py 4096 16384 2>&1
