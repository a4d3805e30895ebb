"""Summarise an ncu launch list (gpu__time_duration.sum) of bench.py: the decode step's kernels only
(each per-token quantizer launch at grid (M,1,1) — plain, or fused into RMSNorm / SiLU·mul in the
fused_block step — and the W4A8 GEMM launch that follows it).

  python tools/launch_share.py gpurun_out/launches.csv [M]
"""
import csv
import sys
from collections import defaultdict


def main(path, M=64):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[i]
    col = {h: hdr.index(h) for h in ("Kernel Name", "Grid Size", "Block Size", "Metric Value")}
    launches = [(r[col["Kernel Name"]], r[col["Grid Size"]], r[col["Block Size"]], float(r[col["Metric Value"]].replace(",", "")))
                for r in rows[i + 1:] if len(r) > col["Metric Value"]]
    t = defaultdict(list)
    for a, b in zip(launches, launches[1:]):
        q = next((n for n in ("quantize_act_kernel", "rmsnorm_quant_kernel", "silu_mul_quant_kernel") if n in a[0]), None)
        if q and a[1] == f"({M}, 1, 1)" and "w4a8_gemm_kernel" in b[0]:
            t[q].append(a[3])
            t[f"w4a8_gemm_kernel grid {b[1]} block {b[2]}"].append(b[3])
    tot = sum(sum(v) for v in t.values())
    print(f"decode-step launches (M={M}), ncu serialized cold-cache times:")
    print(f"{'kernel':60s} {'launches':>8s} {'mean us':>8s} {'share':>6s}")
    for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:60s} {len(v):8d} {sum(v) / len(v) / 1e3:8.2f} {100 * sum(v) / tot:5.1f}%")
    g = sum(sum(v) for k, v in t.items() if k.startswith("w4a8"))
    print(f"{'W4A8 GEMM total share':60s} {'':8s} {'':8s} {100 * g / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 64)
