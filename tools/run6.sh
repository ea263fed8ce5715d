timeout 300 ncu --set full --import-source on --clock-control none -k regex:panel_leaf -s 4 -c 1 -o gpurun_out/prof_leaf512 ./tools/bench_panel_nt > gpurun_out/ncu6a.log 2>&1; echo rc=$?
timeout 300 ncu --set full --import-source on --clock-control none -k regex:panel_leaf -s 19 -c 1 -o gpurun_out/prof_leaf16k ./tools/bench_panel_nt > gpurun_out/ncu6b.log 2>&1; echo rc=$?
