#!/bin/bash
# One gpurun call: GPU tests, smoke, bench line, launch list and one full ncu capture
# of the fused pass.  Usage: gpurun --timeout 2400 -- 'bash tools/gpu_round.sh TAG'
tag=${1:-run}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi > $out/nvidia-smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $out/pytest_gpu.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > $out/smoke.log 2>&1
echo "smoke exit $?" >> $out/smoke.log
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err
echo "bench exit $?" >> $out/bench.err
# launch list (cold-cache, serialised) of a short cfg2 ingestion, then the top kernel in full
cmd="python tools/profile_isvd.py --cols 40"
timeout 600 $cmd > $out/plain.log 2>&1 &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file $out/launches.csv $cmd > $out/ncu_launch.log 2>&1
cmd2="python tools/profile_isvd.py --cols 8"
timeout 600 $cmd2 > $out/plain2.log 2>&1 &&
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_pass -s 230 -c 3 \
    -o $out/pass $cmd2 > $out/ncu_full.log 2>&1
echo done > $out/done
