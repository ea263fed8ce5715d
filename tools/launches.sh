#!/bin/bash
# usage: tools_launches.sh <tag> <bench args...>   (runs plain, then the ncu launch list)
tag=$1; shift
C="python bench.py $@"
$C > gpurun_out/plain_$tag.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv $C > gpurun_out/ncu_$tag.log 2>&1
echo "launches_$tag rc=$?"
