rm -f gpurun_out/timeline.txt; MP_TIMELINE=gpurun_out/timeline.txt timeout 300 python tools/probe_scaling.py 16384 > gpurun_out/tl_probe.log 2>&1
python tools/timeline2.py gpurun_out/timeline.txt
cat gpurun_out/tl_probe.log
