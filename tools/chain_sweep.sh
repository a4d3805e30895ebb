#!/bin/bash
# A/B of the decode chain: k-split cap (QOQ_CHAIN_SMAX) x library variants (ring depths, dequant groups)
cd "$(dirname "$0")/.."
for v in "" x2 g2; do
  for s in 0 1 2; do
    echo "variant=${v:-prod} SMAX=$s"
    QOQ_LIB_VARIANT=$v QOQ_CHAIN_SMAX=$s timeout 120 python tools/chain_bench.py --M 64 --reps 10 2>&1 | tail -1
  done
done
QOQ_CHAIN_SMAX=0 timeout 120 python tools/chain_bench.py --M 1 16 --reps 10 2>&1 | tail -2
