#!/bin/bash
# One `ncu --set full` capture per Llama-3-8B decode GEMM shape (M=64, fused gate_up), for the
# roofline `traffic` field of bench.py. Writes gpurun_out/ncu_<name>.ncu-rep + raw CSVs.
# Reduce with: python tools/ncu_traffic.py gpurun_out > profiles/ncu_traffic.json
set -e
M=${M:-64}
# FUSED=1: the qoq_w4a8_linear kernel (per-token quantization fused into the GEMM)
SUF=""; EXTRA=""
if [ "${FUSED:-0}" = "1" ]; then SUF="_fused"; EXTRA="--fused"; fi
mkdir -p gpurun_out
for spec in qkv:6144:4096 o:4096:4096 gate_up:28672:4096 down:4096:14336; do
  IFS=: read name N K <<< "$spec"
  # skip the first 8 launches (warm-up of the 8 rotating weights), capture 2
  ncu --set full --clock-control none --import-source on -k regex:w4a8_gemm -s 8 -c 2 \
      -o gpurun_out/ncu_${name}_M${M}${SUF} -f \
      python tools/prof_gemm.py --M $M --N $N --K $K --iters 3 --layers 8 $EXTRA > /dev/null
  ncu -i gpurun_out/ncu_${name}_M${M}${SUF}.ncu-rep --page raw --csv > gpurun_out/ncu_${name}_M${M}${SUF}_raw.csv
done
