cd $GRAFT_REPO_ROOT
for b in bench_solve_d2 bench_solve_d1 bench_solve_d2y16 bench_solve_d2y16h12; do echo "== $b"; INV=1 timeout 60 ./tools/$b | tail -3; done
for h in 48 64 80 100; do echo "== d2y16 helpers $h"; MP_SOLVE_HELPERS=$h INV=1 timeout 60 ./tools/bench_solve_d2y16 | tail -1; done
echo "== d2 subst"; timeout 60 ./tools/bench_solve_d2 | tail -1
echo "== d3 subst"; timeout 60 ./tools/bench_solve_nt | tail -1
