#!/bin/bash
# Round-2 GPU call: GPU tests (incl. full-size cfg2 parity), smoke, bench line.
# Usage: gpurun --timeout 3000 -- 'bash tools/gpu_r2.sh TAG [pytest-args]'
tag=${1:-run}
shift
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi > $out/nvidia-smi.txt 2>&1
nproc > $out/nproc.txt; free -g >> $out/nproc.txt; lscpu >> $out/nproc.txt
timeout 1500 python -m pytest tests -m gpu -x -q -s --durations=30 "$@" > $out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $out/pytest_gpu.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > $out/smoke.log 2>&1
echo "smoke exit $?" >> $out/smoke.log
timeout 1200 python bench.py > $out/bench.json 2> $out/bench.err
echo "bench exit $?" >> $out/bench.err
echo done > $out/done
