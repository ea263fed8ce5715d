cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 300 python tools/probe_scaling.py 16384 2>&1 | tail -1
timeout 300 python tools/probe_scaling.py 16384 4096 --noprof 2>&1 | tail -2
