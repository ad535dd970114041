#!/bin/bash
out=gpurun_out/${1:-spdbg}; mkdir -p $out
timeout 120 python -m pytest tests/test_gpu_spatial.py tests/test_gpu_operators.py -q -x > $out/pytest.log 2>&1; echo "exit $?" >> $out/pytest.log
for m in 0 1 2 3; do
  echo "dbg $m: $(STROM_SPATIAL_DBG=$m timeout 90 python tools/st_build.py cm 5 2>&1 | tail -1)" >> $out/log.txt
done
cmd="python tools/st_build.py cm 4"
timeout 90 $cmd > $out/plain.log 2>&1 &&
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spatial_ell -s 2 -c 1 -o $out/sp $cmd > $out/ncu.log 2>&1
