#!/bin/bash
# ncu captures of the kernels changed after tools/gpu_prof_r2.sh's last run: the compaction sweep
# (whole tiles at cfg2) and the tridiagonal FOM march.  Usage: gpurun -- 'bash tools/gpu_prof_extra.sh TAG'
tag=${1:-prof_extra}
out=gpurun_out/$tag
mkdir -p $out
run() {  # name, kernel regex, skip, count, command...
  local name=$1 rx=$2 skip=$3 cnt=$4; shift 4
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s $skip -c $cnt \
      -o $out/$name "$@" > $out/ncu_$name.log 2>&1
  echo "$name rc=$?" >> $out/status.txt
  python tools/ncu_summary.py $out/$name.ncu-rep > $out/sum_$name.txt 2>&1
  python tools/ncu_stalls.py $out/$name.ncu-rep "$rx" > $out/stalls_$name.txt 2>&1
  rm -f $out/$name.ncu-rep
}
timeout 600 python tools/profile_isvd.py --cols 150 > $out/plain_isvd.log 2>&1 &&
  run compact 'k_compact' 0 4 python tools/profile_isvd.py --cols 150
timeout 600 python tools/cfg1_pipeline.py > $out/plain_cfg1.log 2>&1 &&
  run tridiag 'k_fom_tridiag' 4 1 python tools/cfg1_pipeline.py
echo done > $out/done
