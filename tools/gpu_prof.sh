#!/bin/bash
# One gpurun call: full ncu captures of the fused pass (steady-state cfg2) and of the
# cfg4 spatial reduction.  Usage: gpurun -- 'bash tools/gpu_prof.sh TAG'
tag=${1:-prof}
out=gpurun_out/$tag
mkdir -p $out
cmd="python tools/profile_isvd.py --cols 12"
timeout 600 $cmd > $out/plain.log 2>&1 &&
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_pass -s 205 -c 3 \
    -o $out/pass $cmd > $out/ncu_pass.log 2>&1
cmd2="python tools/st_build.py cm 3"
timeout 600 $cmd2 > $out/plain2.log 2>&1 &&
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_spatial -s 2 -c 2 \
    -o $out/spatial $cmd2 > $out/ncu_spatial.log 2>&1
echo done > $out/done
