python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 3 --warmup 3 --variant 3xtf32 --no-cpu --e2e-steps 0 > gpurun_out/bench_tf32.log 2>&1; echo "bench tf32 rc=$?"
tail -c 3000 gpurun_out/bench_tf32.log
