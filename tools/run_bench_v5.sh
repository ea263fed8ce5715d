timeout 600 python bench.py > gpurun_out/bench_v5.json 2> gpurun_out/bench_v5.err; echo bench rc=$?
tail -c 1500 gpurun_out/bench_v5.json
MP_NO_LOOKAHEAD=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v5.csv python bench.py --steps 1 --warmup 1 --fp64-steps 0 --e2e-steps 0 --no-cpu > gpurun_out/ncu_v5.log 2>&1; echo ncu rc=$?
python tools/summarize.py gpurun_out/launches_v5.csv > gpurun_out/launches_v5.txt; head -12 gpurun_out/launches_v5.txt
