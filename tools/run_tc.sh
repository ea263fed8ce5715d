timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for i in 1 2; do timeout 300 python tools/probe_scaling.py 16384 --noprof 2>&1 | tail -1; MP_NO_TC_INPANEL=1 timeout 300 python tools/probe_scaling.py 16384 --noprof 2>&1 | tail -1; done
