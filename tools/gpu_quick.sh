#!/bin/bash
# Quick GPU check: selected tests + one bench line.  Usage: gpurun -- 'bash tools/gpu_quick.sh TAG "pytest args" "bench args"'
tag=${1:-quick}
out=gpurun_out/$tag
mkdir -p $out
timeout 1200 python -m pytest -q -s -x $2 > $out/pytest.log 2>&1
echo "pytest exit $?" >> $out/pytest.log
timeout 900 python bench.py $3 > $out/bench.json 2> $out/bench.err
echo "bench exit $?" >> $out/bench.err
echo done > $out/done
