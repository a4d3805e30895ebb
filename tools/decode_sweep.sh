#!/bin/bash
# timing sweep of the decode GEMMs (Llama-3-8B shapes) — run on the GPU box
for M in 1 16 64 128 256; do
  for NK in "6144 4096" "4096 4096" "14336 4096" "4096 14336"; do
    set -- $NK
    python tools/prof_gemm.py --M $M --N $1 --K $2 --layers 16 --iters 10 --time
  done
done
