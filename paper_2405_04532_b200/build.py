"""Build libqoq_b200.so in-tree with nvcc for sm_100a (the only target)."""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libqoq_b200.so")


def lib_path(variant: str = "") -> str:
    return LIB if not variant else os.path.join(HERE, f"libqoq_b200_{variant}.so")
SOURCES = ["qoq_api.cu", "quantize.cu", "fused_quant.cu", "kv4_attention.cu", "w4a8_gemm.cu", "w4a8_chain.cu"]
HEADERS = ["qoq_internal.h", "sm100_ptx.cuh", "qoq_quant.cuh", "w4a8_common.cuh", os.path.join("..", "..", "include", "qoq_b200.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-cudart", "static", "--expt-relaxed-constexpr"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [os.path.abspath(__file__)]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, extra: list[str] | None = None, variant: str = "") -> str:
    """variant != "": a debug/ablation build (e.g. extra=["-DQOQ_ABLATE=1"]) into libqoq_b200_<variant>.so."""
    out = lib_path(variant)
    if not force and not variant and not _stale():
        return LIB
    objs, cmds = [], []
    for s in SOURCES:
        o = os.path.join(CSRC, s.replace(".cu", f"{variant}.o"))
        cmds.append([NVCC, *FLAGS, *(extra or []), "-c", os.path.join(CSRC, s), "-o", o])
        if verbose:
            print(" ".join(cmds[-1]), file=sys.stderr)
        objs.append(o)
    # translation units compile in parallel (the GEMM and chain files dominate)
    with ThreadPoolExecutor(max_workers=len(cmds)) as ex:
        for f in [ex.submit(subprocess.check_call, c) for c in cmds]:
            f.result()
    tmp = out + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
                           "-o", tmp, *objs, "-lcuda" if False else "-ldl"])
    os.replace(tmp, out)
    for o in objs:
        os.remove(o)
    return out


if __name__ == "__main__":
    extra = ["-Xptxas", "-v"] if "--ptxas" in sys.argv else []
    variant = ""
    for a in sys.argv[1:]:
        if a.startswith("--variant="):   # --variant=name:-DFOO=1,-DBAR=2
            name, flags = a.split("=", 1)[1].split(":", 1)
            variant = name
            extra += flags.split(",")
        if a.startswith("--ablate="):
            variant = "ablate" + a.split("=")[1]
            extra.append("-DQOQ_ABLATE=" + a.split("=")[1])
    print(build(force="--force" in sys.argv or bool(variant), verbose=True, extra=extra, variant=variant))
