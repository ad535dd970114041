#!/bin/bash
# U slack between compactions vs throughput (diagnostics)
for sl in 16 24 32 40 48 63; do
  v=$(STROM_SLACK=$sl timeout 120 python bench.py --skip-st --no-e2e --no-cpu-baseline --steps 3 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('%.0f pass %.1f ms compact %s' % (l['value'], l['kernels']['fused_pass']['ms'], l['kernels'].get('compact_sweep',{}).get('launches')))")
  echo "slack $sl : $v"
done
