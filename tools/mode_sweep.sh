#!/bin/bash
# planner-mode comparison (0: whole tiles, 1: stream-K + L2 workspace, 2: cluster DSMEM split-K)
for M in 16 64; do
  for NK in "6144 4096" "4096 4096" "14336 4096" "4096 14336" "28672 4096"; do
    set -- $NK
    for mode in 0 1 2; do echo -n "mode $mode: "; QOQ_FORCE_MODE=$mode python tools/prof_gemm.py --M $M --N $1 --K $2 --layers 16 --iters 10 --time; done
  done
done
