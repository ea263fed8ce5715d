cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for i in 1 2; do
timeout 300 python tools/probe_scaling.py 16384 8192 --noprof 2>&1 | tail -2
MP_NO_LA_SPLIT=1 timeout 300 python tools/probe_scaling.py 16384 8192 --noprof 2>&1 | tail -2
done
