cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "exchange or deterministic" 2>&1 | tail -3
for e in "X=0" "MP_PANEL_SMS=40" "MP_PANEL_SMS=56" "MP_PANEL_SMS_EARLY=24" "MP_PANEL_SMS_EARLY=40" "MP_EARLY_FRAC=0.6" "MP_FUSED_GRID=128"; do
  echo "== $e"; env $e timeout 300 python tools/probe_scaling.py 16384 --noprof 2>&1 | tail -1 | cut -c1-90
done
