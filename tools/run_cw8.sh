cd $GRAFT_REPO_ROOT
MP_TRSM_CW=8 timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for i in 1 2; do
for c in 16 8; do echo "cw $c"; MP_TRSM_CW=$c timeout 300 python tools/probe_scaling.py 16384 4096 --noprof 2>&1 | tail -2 | cut -c1-100; done
done
