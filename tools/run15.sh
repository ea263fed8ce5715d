timeout 300 python tools/probe_scaling.py 16384 --noprof 2>&1
timeout 300 python tools/probe_scaling.py 16384 2>&1
