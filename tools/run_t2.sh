timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for i in 1 2; do timeout 300 python tools/probe_scaling.py 16384 --noprof 2>&1 | tail -1 | cut -c1-90; done
bash tools/run_tl.sh 2>&1 | grep -E "panel stream|update stream"
