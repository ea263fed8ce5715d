cd $GRAFT_REPO_ROOT
for e in "" "NOTAGS=1"; do echo "== $e"; env INV=1 $e timeout 120 ./tools/bench_solve_nt; done
echo "== trace"; INV=1 timeout 120 ./tools/bench_solve | tail -6
timeout 900 python -m pytest tests -m gpu -x -q -k "solve or parity or many_rhs or inv" 2>&1 | tail -3
MP_SOLVE_FLAGS=1 timeout 300 python tools/probe_scaling.py 2>&1 | tail -4
timeout 300 python tools/probe_scaling.py 2>&1 | tail -4
