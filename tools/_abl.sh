for M in 64 16; do
for NK in "28672 4096" "4096 4096"; do
  set -- $NK
  echo -n "M=$M base     "; python tools/prof_gemm.py --M $M --N $1 --K $2 --layers 16 --iters 10 --time
  for a in 16 4 20 32 6; do echo -n "M=$M ablate$a "; QOQ_LIB_VARIANT=ablate$a python tools/prof_gemm.py --M $M --N $1 --K $2 --layers 16 --iters 10 --time; done
done; done
