#!/bin/bash
# compare the production library with a variant build on the decode shapes: tools/variant_sweep.sh <variant>
V=$1
for M in 16 64; do
  for NK in "6144 4096" "4096 4096" "28672 4096" "4096 14336"; do
    set -- $NK
    echo -n "base : "; python tools/prof_gemm.py --M $M --N $1 --K $2 --layers 16 --iters 10 --time
    echo -n "$V: "; QOQ_LIB_VARIANT=$V python tools/prof_gemm.py --M $M --N $1 --K $2 --layers 16 --iters 10 --time
  done
done
