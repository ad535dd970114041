#!/bin/bash
# Round-2 ncu captures of every hot-path kernel (one capture each, after the
# plain command has exited 0).  Usage: gpurun -- 'bash tools/gpu_prof_r2.sh TAG'
tag=${1:-prof}
out=gpurun_out/$tag
mkdir -p $out
run() {  # name, kernel regex, skip, count, command...
  local name=$1 rx=$2 skip=$3 cnt=$4; shift 4
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s $skip -c $cnt \
      -o $out/$name "$@" > $out/ncu_$name.log 2>&1
  echo "$name rc=$?" >> $out/status.txt
  # summaries on the box (the reports themselves exceed gpurun's copy-back cap)
  python tools/ncu_summary.py $out/$name.ncu-rep > $out/sum_$name.txt 2>&1
  python tools/ncu_stalls.py $out/$name.ncu-rep "$rx" > $out/stalls_$name.txt 2>&1
  ncu -i $out/$name.ncu-rep --page details --csv > $out/details_$name.csv 2>/dev/null
  rm -f $out/$name.ncu-rep
}
timeout 600 python tools/profile_isvd.py --cols 150 > $out/plain_isvd.log 2>&1 && {
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
      --log-file $out/launches_isvd.csv python tools/profile_isvd.py --cols 40 > $out/ncu_launch.log 2>&1
  run step_b 'k_step_b' 110 2 python tools/profile_isvd.py --cols 40
  run decide 'k_decide' 330 4 python tools/profile_isvd.py --cols 40
  run vupdate 'k_vupdate' 110 2 python tools/profile_isvd.py --cols 40
  run pass 'k_pass' 120 4 python tools/profile_isvd.py --cols 40
  run wproj 'k_wproj' 14 2 python tools/profile_isvd.py --cols 40
  run compact 'k_compact' 0 4 python tools/profile_isvd.py --cols 150
}
timeout 600 python tools/prof_targets.py st 2 > $out/plain_st.log 2>&1 && {
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file $out/launches_st.csv python tools/prof_targets.py st 1 > $out/ncu_launch_st.log 2>&1
  run st_kernels 'k_st_|k_spatial_ell' 6 6 python tools/prof_targets.py st 2
  run lu 'k_lu_persistent' 0 1 python tools/prof_targets.py st 1
  run reconstruct 'k_reconstruct' 0 1 python tools/prof_targets.py st 1
}
timeout 600 python tools/prof_targets.py cfg1 2 > $out/plain_cfg1.log 2>&1 && \
  run small_svd 'k_small_svd' 0 1 python tools/prof_targets.py cfg1 1
echo done > $out/done
