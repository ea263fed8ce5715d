timeout 600 python bench.py > gpurun_out/bench_v13.json 2> gpurun_out/bench_v13.err; echo bench rc=$?
tail -1 gpurun_out/bench_v13.json | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['speedup_vs_fp64'], d['e2e']['ms_per_step'], d['roofline']['frac'], d['panel_us_per_column'], d['clocks'])"
MP_NO_LOOKAHEAD=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v13.csv python bench.py --steps 1 --warmup 1 --fp64-steps 0 --e2e-steps 0 --no-cpu > gpurun_out/ncu_v13.log 2>&1; echo ncu rc=$?
python tools/summarize.py gpurun_out/launches_v13.csv > gpurun_out/launches_v13.txt; head -14 gpurun_out/launches_v13.txt
