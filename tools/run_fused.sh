timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_fused.log 2>&1; tail -30 gpurun_out/pytest_fused.log | grep -E "passed|failed|Error|assert" | head -20
for i in 1 2; do timeout 300 python tools/probe_scaling.py 16384 --noprof 2>&1 | tail -1; MP_NO_FUSED_TRSM=1 timeout 300 python tools/probe_scaling.py 16384 --noprof 2>&1 | tail -1; done
