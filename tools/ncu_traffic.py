"""Reduce the raw CSVs of tools/ncu_traffic.sh to profiles/ncu_traffic.json.

For each shape: dram__bytes_read.sum + dram__bytes_write.sum per launch (mean over captured launches);
the bench key "<model>-M<M>" holds the mean over the step's four GEMM shapes (each launched once
per layer, so the mean is the per-launch figure bench.py's `achieved` is computed on).
"""
import csv
import glob
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import gemm_bytes  # noqa: E402

SHAPES = {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (28672, 4096), "down": (4096, 14336)}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def launches(path):
    with open(path) as f:
        rows = list(csv.reader(f))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        tot = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            tot += float(d[m].replace(",", "")) * UNIT[u[m]]
        out.append(tot)
    return out


def main(src):
    res = {}
    for name, (N, K) in SHAPES.items():
        for p in glob.glob(os.path.join(src, f"ncu_{name}_M*_raw.csv")):
            tag = os.path.basename(p)[len(f"ncu_{name}_M"):-len("_raw.csv")]   # "64" or "64_fused"
            M = int(tag.split("_")[0])
            key = f"llama3-8b-M{M}" + ("-fused" if tag.endswith("_fused") else "")
            v = launches(p)
            res.setdefault(key, {})[name] = {"dram_bytes_per_launch": sum(v) / len(v),
                                             "algorithmic_bytes": gemm_bytes(M, N, K), "launches": len(v)}
    out = {}
    for key, d in sorted(res.items()):
        if len(d) == len(SHAPES):
            out[key] = sum(x["dram_bytes_per_launch"] for x in d.values()) / len(d)
        out[key + "-shapes"] = d
    out["source"] = ("ncu --set full --clock-control none (tools/ncu_traffic.sh), "
                     "dram__bytes_read.sum + dram__bytes_write.sum")
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out")
