timeout 300 python tools/probe_scaling.py 16384 2>&1
MP_NO_LOOKAHEAD=1 timeout 300 python tools/probe_scaling.py 16384 2>&1
