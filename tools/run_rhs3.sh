cd $GRAFT_REPO_ROOT
timeout 600 python tools/probe_rhs.py 2>&1 | tail -3
