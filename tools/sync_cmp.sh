#!/bin/bash
for d in 0 1 2 3; do
  v=$(STROM_SYNC_DEBUG=$d timeout 120 python bench.py --skip-st --no-e2e --no-cpu-baseline --steps 5 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=l['kernels']; print('%.0f' % l['value'])")
  echo "sync_debug $d : $v"
done
