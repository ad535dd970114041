#!/bin/bash
# cfg3 iSVD throughput in window mode vs the per-snapshot mode, plus an uncapped trace
out=gpurun_out/$1; mkdir -p $out
python tools/cfg3_transport.py > $out/cfg3_window.json 2>&1
STROM_WINDOW=1 python tools/cfg3_transport.py > $out/cfg3_old.json 2>&1
python tools/trace_isvd.py --uncapped --tol 1e-8 > $out/trace_uncapped.txt 2>&1
