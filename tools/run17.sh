python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/probe_scaling.py 4096 16384 --noprof 2>&1
MP_NO_LOOKAHEAD=1 timeout 300 python tools/probe_scaling.py 16384 --noprof 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
