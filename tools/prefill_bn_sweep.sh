#!/bin/bash
# Prefill token-tile sweep: TOPS per Llama-3-8B GEMM at M = 1024 / 2048 / 4096 for the planner's choice and each
# forced token tile (QOQ_BN_BIG = 128 / 192 / 256).
for M in ${MS:-1024 2048 4096}; do
for NK in "6144 4096" "4096 4096" "28672 4096" "4096 14336"; do set -- $NK
  line="M=$M N=$1 K=$2:"
  for bn in 0 128 192 256; do
    r=$(QOQ_BN_BIG=$bn timeout 120 python tools/prof_gemm.py --M $M --N $1 --K $2 --layers 4 --iters 5 --time 2>&1 | grep -o "[0-9.]* TOPS")
    line="$line bn=$bn ${r}"
  done
  echo "$line"
done; done
