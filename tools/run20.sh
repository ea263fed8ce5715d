python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python bench.py --dist --steps 2 --warmup 1 --no-cpu --e2e-steps 1 --fp64-steps 1 2>&1 | tail -c 1500
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --dist --steps 2 --warmup 1 --no-cpu --e2e-steps 0 --fp64-steps 0 --n 8192 2>&1 | tail -c 800
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
