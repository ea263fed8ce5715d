cd $GRAFT_REPO_ROOT
for b in bench_solve_nt bench_solve_d2 bench_solve_d2c3 bench_solve_yb4 bench_solve_yb16; do echo "== $b"; INV=1 timeout 60 ./tools/$b | tail -1; done
for h in 32 64 100; do echo "== helpers $h"; MP_SOLVE_HELPERS=$h INV=1 timeout 60 ./tools/bench_solve_nt | tail -1; done
