#!/bin/bash
# One gpurun call: cfg1/cfg3 pipelines and a full ncu capture of the single-CTA
# fom_march.  Usage: gpurun -- 'bash tools/gpu_fom.sh TAG'
out=gpurun_out/${1:-fom}; mkdir -p $out
timeout 300 python tools/cfg1_pipeline.py > $out/cfg1.json 2> $out/cfg1.err; echo "cfg1 exit $?" >> $out/cfg1.err
timeout 600 python tools/cfg3_transport.py > $out/cfg3.json 2> $out/cfg3.err; echo "cfg3 exit $?" >> $out/cfg3.err
cmd="python tools/fom_profile.py 0"
timeout 120 $cmd > $out/fom_plain.log 2>&1 &&
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fom_march -s 1 -c 1 \
    -o $out/fom $cmd > $out/fom_ncu.log 2>&1
