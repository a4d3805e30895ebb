#!/bin/bash
# prefill (tensor-bound) token-tile A/B: planner choice vs forced BN = 128 / 192 / 256
for M in ${MS:-1024 4096 8192}; do
  for NK in "6144 4096" "4096 4096" "28672 4096" "4096 14336"; do
    set -- $NK
    for cfg in "" "QOQ_BN_BIG=128" "QOQ_BN_BIG=192" "QOQ_BN_BIG=256"; do
      echo -n "[${cfg:-auto}] "; env $cfg python tools/prof_gemm.py --M $M --N $1 --K $2 --layers 4 --iters 5 --time 2>&1 | tail -1
    done
  done
done
