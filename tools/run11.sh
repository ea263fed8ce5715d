rm -f gpurun_out/timeline.txt; MP_TIMELINE=gpurun_out/timeline.txt timeout 300 python tools/probe_scaling.py 16384 > /dev/null 2>&1
python tools/timeline.py gpurun_out/timeline.txt
timeout 300 python tools/probe_scaling.py 16384 > gpurun_out/plain11.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches11.csv python tools/probe_scaling.py 16384 > gpurun_out/ncu11.log 2>&1; echo ncu rc=$?
python tools/summarize.py gpurun_out/launches11.csv
