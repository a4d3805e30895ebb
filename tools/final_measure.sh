#!/bin/bash
# Round-end measurement set (one GPU): full GPU suite, default bench line, ncu launch list of the decode step
# and its share, one ncu --set full capture per decode GEMM shape (roofline traffic).
cd "$(dirname "$0")/.."
P=${1:-r2b}
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${P}_pytest_gpu.log 2>&1
tail -3 gpurun_out/${P}_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/${P}_bench.json 2> gpurun_out/${P}_bench.err
tail -2 gpurun_out/${P}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1400 --csv --log-file gpurun_out/${P}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-prefill --no-e2e --no-cpu-baseline --no-fused-block --no-kv4 --no-per-channel \
  --no-chain --no-sweep --no-tp-fused > /dev/null 2>&1
python tools/launch_share.py gpurun_out/${P}_launches.csv > gpurun_out/${P}_launch_share.txt 2>&1
timeout 1200 bash tools/ncu_traffic.sh > /dev/null 2>&1
python tools/ncu_traffic.py gpurun_out > gpurun_out/${P}_ncu_traffic.json 2>&1
cat gpurun_out/${P}_launch_share.txt
