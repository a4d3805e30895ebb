"""Run the NEXT-2 fused quantizers once per shape (for ncu captures; no timing here).

  python tools/prof_fused.py --M 4096 [--kind rms|silu|both]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2405_04532_b200 as qoq  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=4096)
    ap.add_argument("--K", type=int, default=4096)
    ap.add_argument("--I", type=int, default=14336)
    ap.add_argument("--kind", default="both")
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    qoq.load()
    gen = torch.Generator(device=dev)
    gen.manual_seed(1)
    X = synth.device_activations_fp16(a.M, a.K, gen, dev)
    g = (1.0 + 0.1 * torch.randn(a.K, generator=gen, device=dev)).half()
    GU = (2.0 * torch.randn(a.M, 2 * a.I, generator=gen, device=dev)).half()
    for _ in range(a.reps):
        if a.kind in ("rms", "both"):
            qoq.rmsnorm_quantize(X, g, 1e-5)
        if a.kind in ("silu", "both"):
            qoq.silu_mul_quantize(GU)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
