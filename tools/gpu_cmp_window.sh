#!/bin/bash
# iSVD parity tests in window mode and in per-snapshot mode (STROM_WINDOW=1), no -x.
out=gpurun_out/$1
mkdir -p $out
timeout 900 python -m pytest -q -s tests/test_gpu_isvd.py tests/test_gpu_capacity.py tests/test_gpu_cfg2_full.py tests/test_gpu_basis_mirror.py -m gpu > $out/win.log 2>&1
echo "exit $?" >> $out/win.log
STROM_WINDOW=1 timeout 900 python -m pytest -q -s tests/test_gpu_capacity.py tests/test_gpu_cfg2_full.py -m gpu > $out/old.log 2>&1
echo "exit $?" >> $out/old.log
STROM_WINDOW=1 python tools/profile_isvd.py --cols 120 > $out/old_counts.txt 2>&1
python tools/profile_isvd.py --cols 120 > $out/win_counts.txt 2>&1
