#!/bin/bash
# timing ablations of the W4A8 GEMM mainloop (QOQ_ABLATE bits in w4a8_gemm.cu); run on the GPU box
for a in 2 4 8 14; do python paper_2405_04532_b200/build.py --ablate=$a > /dev/null 2>&1; done
for NK in "28672 4096" "4096 4096"; do
  set -- $NK
  echo -n "base     "; python tools/prof_gemm.py --M 64 --N $1 --K $2 --layers 16 --iters 10 --time
  for a in 2 4 8 14; do echo -n "ablate$a "; QOQ_LIB_VARIANT=ablate$a python tools/prof_gemm.py --M 64 --N $1 --K $2 --layers 16 --iters 10 --time; done
done
