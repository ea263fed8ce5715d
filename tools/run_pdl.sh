timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_pdl.log 2>&1; tail -3 gpurun_out/pytest_pdl.log
for i in 1 2; do
timeout 300 python tools/probe_scaling.py 16384 --noprof 2>&1 | tail -1
MP_NO_PDL=1 timeout 300 python tools/probe_scaling.py 16384 --noprof 2>&1 | tail -1
done
