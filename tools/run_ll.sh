timeout 300 python tools/probe_scaling.py 16384 --noprof > gpurun_out/ll_plain.log 2>&1 && MP_NO_LOOKAHEAD=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll.csv python tools/probe_scaling.py 16384 --noprof > gpurun_out/ll_ncu.log 2>&1; echo ncu rc=$?
python tools/summarize.py gpurun_out/ll.csv | head -25
cat gpurun_out/ll_plain.log
