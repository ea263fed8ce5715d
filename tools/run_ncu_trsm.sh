cd $GRAFT_REPO_ROOT
MP_NO_LOOKAHEAD=1 timeout 120 python tools/probe_scaling.py 8192 --noprof > /dev/null 2>&1 && echo pre-ok
MP_NO_LOOKAHEAD=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:trsm_lower_unit -s 54 -c 8 -o gpurun_out/prof_trsm2 python tools/probe_scaling.py 8192 --noprof > gpurun_out/ncu_trsm2.log 2>&1; echo rc=$?
