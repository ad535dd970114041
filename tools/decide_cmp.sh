#!/bin/bash
for d in 0 1; do
  v=$(STROM_DECIDE_KERNEL=$d timeout 120 python bench.py --skip-st --no-e2e --no-cpu-baseline --steps 3 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=l['kernels']; print('%.0f pass %.1f step_a %s' % (l['value'], k['fused_pass']['ms'], k.get('step_a',{}).get('ms')))")
  echo "decide_kernel $d : $v"
done
