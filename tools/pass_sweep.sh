#!/bin/bash
# pass bandwidth probes on the bench workload (diagnostics; values of a dbg run are not results)
for d in 0 1; do for kb in 60 100 140 200; do
  v=$(STROM_PASS_DBG=$d STROM_STAGE_KB=$kb timeout 120 python bench.py --skip-st --no-e2e --no-cpu-baseline --steps 3 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('%.0f %.0f' % (l['value'], l['kernels']['fused_pass']['gbs']))")
  echo "dbg $d stage_kb $kb : $v"
done; done
