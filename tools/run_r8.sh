cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 600 python tools/probe_rhs.py 2>&1 | tail -4
