#!/bin/bash
out=gpurun_out/${1:-spdbg}; mkdir -p $out
timeout 120 python -m pytest tests/test_gpu_spatial.py tests/test_gpu_operators.py -q -x > $out/pytest.log 2>&1; echo "exit $?" >> $out/pytest.log
echo "$(timeout 90 python tools/st_build.py cm 6 2>&1 | tail -1)" >> $out/log.txt
cmd="python tools/st_build.py cm 4"
timeout 90 $cmd > $out/plain.log 2>&1 &&
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv $cmd > $out/ncu.log 2>&1
