#!/bin/bash
# spatial-reduction iteration: parity tests, cfg4 build timing, ncu of the spatial kernel
tag=${1:-sp}
out=gpurun_out/$tag
mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_spatial.py tests/test_gpu_operators.py -x -q > $out/pytest.log 2>&1
echo "exit $?" >> $out/pytest.log
cmd="python tools/st_build.py cm 8"
timeout 600 $cmd > $out/plain.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spatial -s 4 -c 2 \
    -o $out/spatial $cmd > $out/ncu.log 2>&1
echo done > $out/done
