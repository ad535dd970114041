#!/bin/bash
out=gpurun_out/${1:-cfg5}; mkdir -p $out
timeout 300 python tools/cfg5_capacity.py --log2n 20 --cols 300 > $out/small.json 2> $out/small.err
echo "small exit $?" >> $out/small.err
timeout 900 python tools/cfg5_capacity.py > $out/full.json 2> $out/full.err
echo "full exit $?" >> $out/full.err
nvidia-smi --query-gpu=memory.total,memory.used --format=csv >> $out/full.err
