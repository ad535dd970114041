#!/bin/bash
# bench line + launch list of the cfg4 build (ncu) for the round's profiles
tag=${1:-bench}
out=gpurun_out/$tag
mkdir -p $out
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err
echo "bench exit $?" >> $out/bench.err
cmd="python tools/st_build.py cm 4"
timeout 120 $cmd > $out/plain.log 2>&1 &&
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/st_launches.csv $cmd > $out/ncu.log 2>&1
timeout 120 $cmd > $out/plain2.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spatial_ell -s 2 -c 1 -o $out/spatial $cmd > $out/ncu2.log 2>&1
