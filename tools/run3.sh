python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/probe_scaling.py 1024 2048 4096 8192 16384 2>&1 | tee gpurun_out/probe_scaling.log
rm -f gpurun_out/timeline.txt; MP_TIMELINE=gpurun_out/timeline.txt timeout 300 python tools/probe_scaling.py 16384 > /dev/null 2>&1
timeout 120 ./tools/probe_green 2>&1 | tee gpurun_out/probe_green.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:panel_leaf -s 40 -c 2 -o gpurun_out/prof_panel python tools/probe_scaling.py 16384 > gpurun_out/ncu_panel.log 2>&1; echo "ncu rc=$?"
