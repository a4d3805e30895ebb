#!/bin/bash
# compute-sanitizer over every kernel family (tools/sanitize_cases.py), one tool at a time, each case in
# its own process (a persistent kernel that spins on grid-wide counters needs all CTAs resident).
#   bash tools/sanitize.sh [out_dir]
cd "$(dirname "$0")/.."
OUT=${1:-gpurun_out}
CS=/usr/local/cuda/bin/compute-sanitizer
CASES=${CASES:-gemm_mode0 gemm_mode1 gemm_mode2 gemm_cg2 gemm_prefill fused_linear per_channel quantizers kv4 chain tp_fused}
for tool in memcheck racecheck synccheck initcheck; do
  for c in $CASES; do
    echo "=== $tool $c"
    timeout 600 $CS --tool $tool --print-limit 20 python tools/sanitize_cases.py --case $c 2>&1 | \
      grep -E "ERROR SUMMARY|RACECHECK SUMMARY|case .*: ok|Error|error|Hazard|hazard|Timeout|Killed" | head -20
    echo "rc=${PIPESTATUS[0]}"
  done
done > $OUT/sanitize.txt 2>&1
