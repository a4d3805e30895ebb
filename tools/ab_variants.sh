#!/bin/bash
# A/B of library variants (built with build.py --variant=name:flags) on the decode step + per-GEMM detail.
# usage: tools/ab_variants.sh "M list" variant...   ("" = production build)
Ms=$1; shift
for M in $Ms; do
  for v in "$@"; do
    echo "== M=$M variant=${v:-prod}"
    QOQ_LIB_VARIANT=$v timeout 300 python bench.py --M $M --no-e2e --no-cpu-baseline --no-prefill --detail 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('value %.1f GB/s  ms/step %.3f  gemm frac %.3f' % (d['value'], d['ms_per_step'], d['roofline']['frac']))
print('  ' + '  '.join('%s %.2fus' % (k, v['us']) for k,v in d.get('detail',{}).items() if isinstance(v, dict) and 'us' in v))
"
  done
done
