python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --variant 3xtf32 > gpurun_out/bench14.log 2>&1; echo "bench rc=$?"
tail -c 2500 gpurun_out/bench14.log
timeout 300 python bench.py --steps 1 --warmup 3 --variant 3xtf32 --no-cpu --fp64-steps 0 --e2e-steps 0 > gpurun_out/plain14.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches14.csv python bench.py --steps 1 --warmup 3 --variant 3xtf32 --no-cpu --fp64-steps 0 --e2e-steps 0 > gpurun_out/ncu14.log 2>&1; echo "ncu rc=$?"
python tools/summarize.py gpurun_out/launches14.csv
