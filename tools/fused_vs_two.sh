#!/bin/bash
# per-launch time of qoq_w4a8_linear (fused) vs quantizer + GEMM, Llama-3-8B decode shapes
M=${M:-64}
for spec in 6144:4096 4096:4096 28672:4096 4096:14336; do
  IFS=: read N K <<< "$spec"
  echo "N=$N K=$K  gemm only : $(timeout 60 python tools/prof_gemm.py --M $M --N $N --K $K --time | tail -1)"
  echo "N=$N K=$K  quant+gemm: $(timeout 60 python tools/prof_gemm.py --M $M --N $N --K $K --time --with-quant | tail -1)"
  echo "N=$N K=$K  fused     : $(timeout 60 python tools/prof_gemm.py --M $M --N $N --K $K --time --fused | tail -1)"
done
