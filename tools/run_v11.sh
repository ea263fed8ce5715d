cd $GRAFT_REPO_ROOT
bash tools/run_final11.sh
INV=1 timeout 100 ./tools/bench_solve_nt > /dev/null && INV=1 timeout 300 ncu --set full --import-source on --clock-control none -k regex:tri_sweep -s 10 -c 1 -o gpurun_out/prof_solve_v11 ./tools/bench_solve_nt > gpurun_out/ncu_solve_v11.log 2>&1; echo rc=$?
