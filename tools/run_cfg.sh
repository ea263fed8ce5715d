cd $GRAFT_REPO_ROOT
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 900 python tools/probe_configs.py c5 c4 2>&1 | tail -8 | tee gpurun_out/configs_v12.txt
