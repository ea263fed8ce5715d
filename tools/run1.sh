set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --steps 5 --warmup 3 --variant 3xtf32 > gpurun_out/bench_tf32.log 2>&1; echo "bench tf32 rc=$?"
timeout 600 python bench.py --steps 5 --warmup 3 --variant ffma --no-cpu > gpurun_out/bench_ffma.log 2>&1; echo "bench ffma rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_tf32.csv python bench.py --steps 1 --warmup 3 --variant 3xtf32 --no-cpu --fp64-steps 0 --e2e-steps 0 > gpurun_out/ncu_l.log 2>&1; echo "ncu rc=$?"
