"""Time the per-token activation quantizer alone (graph of launches) for one shape.

  python tools/prof_quant.py --M 64 --K 14336 [--iters 20]
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
    ap.add_argument("--M", type=int, default=64)
    ap.add_argument("--K", type=int, default=4096)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--launches", type=int, default=32)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    qoq.load()
    gen = torch.Generator(device=dev)
    gen.manual_seed(1)
    X = synth.device_activations_fp16(a.M, a.K, gen, dev)
    out = qoq.quantize_activations_per_token(X)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            qoq.quantize_activations_per_token(X, out=out, stream=s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(a.launches):
                qoq.quantize_activations_per_token(X, out=out, stream=s)
        for _ in range(3):
            g.replay()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(a.iters):
            g.replay()
        e1.record(s)
        s.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (a.iters * a.launches)
    print(f"quantize M={a.M} K={a.K}: {us:.2f} us/launch ({3 * a.M * a.K / us / 1e3:.0f} GB/s)")


if __name__ == "__main__":
    main()
