#!/bin/bash
out=gpurun_out/${1:-spdbg}; mkdir -p $out
for c in 1 2 3 4 8; do
  echo "chunk $c: $(STROM_SPATIAL_CHUNK=$c timeout 90 python tools/st_build.py cm 6 2>&1 | tail -1)" >> $out/log.txt
done
STROM_SPATIAL_CHUNK=4 timeout 300 python -m pytest tests/test_gpu_spatial.py -q -x > $out/pytest.log 2>&1; echo "exit $?" >> $out/pytest.log
