#!/bin/bash
# Decode A/B: per-projection GEMM time (graph of 16 layers x 10 iterations, prof_gemm --time) and the full
# decode step (bench.py, decode legs only) for the production library and each variant build.
#   bash tools/ab_decode.sh variant1 variant2 ...   (M from $M, default 64)
M=${M:-64}
Q="--no-prefill --no-e2e --no-cpu-baseline --no-fused-block --no-kv4 --no-per-channel --no-chain --no-sweep --steps 50 --M $M"
for v in "" "$@"; do
  line="variant=${v:-prod} M=$M:"
  for NK in "6144 4096" "4096 4096" "28672 4096" "4096 14336"; do
    set -- $NK
    t=$(QOQ_LIB_VARIANT=$v timeout 120 python tools/prof_gemm.py --M $M --N $1 --K $2 --layers 16 --iters 10 --time 2>/dev/null | grep -o "[0-9.]* us" | head -1)
    line="$line ${1}x${2}=${t}"
  done
  r=$(QOQ_LIB_VARIANT=$v timeout 120 python bench.py $Q 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(f\"step {d['ms_per_step']*1e3:.1f} us gemm {d['roofline']['avg_launch_us']:.2f} us/launch frac {d['roofline']['frac']:.3f}\")")
  echo "$line | $r"
done
