#!/bin/bash
out=gpurun_out/${1:-cfg3}; mkdir -p $out
timeout 300 python -m pytest tests/test_gpu_fom.py -q -x > $out/pytest.log 2>&1; echo "exit $?" >> $out/pytest.log
timeout 600 python tools/cfg3_transport.py --nc 16 > $out/small.json 2> $out/small.err; echo "small exit $?" >> $out/small.err
timeout 900 python tools/cfg3_transport.py > $out/full.json 2> $out/full.err; echo "full exit $?" >> $out/full.err
