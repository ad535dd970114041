#!/bin/bash
for kb in 140 160 200 212; do
  v=$(STROM_STAGE_KB=$kb timeout 120 python bench.py --skip-st --no-e2e --no-cpu-baseline --steps 5 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=l['kernels']; print('%.0f pass_gbs %.0f' % (l['value'], k['fused_pass']['gbs']))")
  echo "stage_kb $kb : $v"
done
