#!/bin/bash
# A/B the production library against variants on the decode bench (no prefill/e2e/cpu legs).
#   bash tools/ab.sh early other ...   (variants built with build.py --variant=NAME:...)
Q="--no-prefill --no-e2e --no-cpu-baseline --no-fused-block --no-kv4 --no-per-channel --steps 50 ${AB_EXTRA}"
for rep in 1 2; do
  for v in "" "$@"; do
    r=$(QOQ_LIB_VARIANT=$v timeout 120 python bench.py $Q 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(f\"{d['value']:.0f} GB/s step {d['ms_per_step']*1e3:.1f} us gemm {d['roofline']['avg_launch_us']:.2f} us/launch\")")
    echo "variant=${v:-prod} M=${M:-64}: $r"
  done
done
