#!/bin/bash
# One parameterised GPU-box script (run via gpurun from the repo root); results land in gpurun_out/.
#   bash tools/gpu.sh tests  [pytest -k expr]     -> pytest -m gpu (log + parity JSON lines)
#   bash tools/gpu.sh bench  <tag> [bench args]   -> plain bench line, then the ncu launch list
#   bash tools/gpu.sh ncu    <tag> <kernel regex> [bench args]  -> one ncu --set full capture
#   bash tools/gpu.sh smoke                        -> __graft_entry__.smoke() + its ncu launch list
set -u
mkdir -p gpurun_out
what=$1; shift
case $what in
tests)
    k=${1:-}
    export MP_PARITY_LOG=gpurun_out/parity.jsonl
    timeout 1800 python -m pytest tests -q -m gpu ${k:+-k "$k"} -s > gpurun_out/pytest.log 2>&1
    echo "pytest rc=$?"; tail -3 gpurun_out/pytest.log ;;
bench)
    tag=$1; shift
    timeout 900 python bench.py "$@" > gpurun_out/bench_$tag.log 2>&1; echo "bench rc=$?"
    tail -1 gpurun_out/bench_$tag.log
    MP_NO_LOOKAHEAD=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches_$tag.csv python bench.py "$@" > gpurun_out/ncu_$tag.log 2>&1
    echo "launches rc=$?" ;;
ncu)
    tag=$1; kre=$2; shift 2
    MP_NO_LOOKAHEAD=1 timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$kre" -c 1 \
        -o gpurun_out/full_$tag python bench.py "$@" > gpurun_out/ncufull_$tag.log 2>&1
    echo "ncu rc=$?" ;;
smoke)
    timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" \
        > gpurun_out/ncu_smoke.log 2>&1; echo "ncu rc=$?" ;;
*)
    echo "unknown: $what"; exit 2 ;;
esac
