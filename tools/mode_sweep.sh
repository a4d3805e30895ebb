#!/bin/bash
# planner-mode comparison (0: whole tiles, 1: stream-K + L2 workspace, 2: cluster DSMEM split-K)
# per decode shape, GEMM-only CUDA graph over 16 distinct weight sets (> L2)
for M in ${MS:-1 16 64}; do
  for NK in "6144 4096" "4096 4096" "28672 4096" "4096 14336"; do
    set -- $NK
    for mode in auto 0 1 2; do
      echo -n "mode $mode: "
      if [ $mode = auto ]; then python tools/prof_gemm.py --M $M --N $1 --K $2 --layers 16 --iters 10 --time
      else QOQ_FORCE_MODE=$mode python tools/prof_gemm.py --M $M --N $1 --K $2 --layers 16 --iters 10 --time; fi
    done
  done
done
