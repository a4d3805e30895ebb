"""Run a few W4A8 GEMM launches of one shape (for ncu captures and quick timing).

  python tools/prof_gemm.py --M 64 --N 4096 --K 4096 [--iters 5] [--layers 8] [--time]

--layers rotates over distinct packed weights (> L2 when large) so HBM traffic is honest.
--time prints CUDA-event timing of a graph of `iters x layers` launches (per-launch us, GB/s, TOPS).
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2405_04532_b200 as qoq  # noqa: E402
import synth  # noqa: E402
from bench import gemm_bytes, gemm_ops  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=64)
    ap.add_argument("--N", type=int, default=4096)
    ap.add_argument("--K", type=int, default=4096)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--time", action="store_true")
    ap.add_argument("--with-quant", action="store_true")
    ap.add_argument("--fused", action="store_true", help="qoq_w4a8_linear (quantization fused into the GEMM)")
    ap.add_argument("--pc", action="store_true", help="per-channel W4A8 (qoq_pc_w4a8_gemm, NEXT-1)")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    qoq.load()
    gen = torch.Generator(device=dev)
    packs = []
    for l in range(a.layers):
        gen.manual_seed(l)
        W = synth.device_weights_fp16(a.N, a.K, gen, dev)
        packs.append(qoq.pc_quantize_weights(W) if a.pc else qoq.quantize_weights(W))
    X = synth.device_activations_fp16(a.M, a.K, gen, dev)
    q = qoq.quantize_activations_per_token(X)
    Y = torch.empty(a.M, a.N, dtype=torch.float16, device=dev)
    ws = qoq.Workspace(dev)
    s = torch.cuda.Stream()

    def run():
        for pk in packs:
            if a.pc:
                qoq.pc_w4a8_gemm(*q, *pk, a.N, out=Y, workspace=ws, stream=s)
                continue
            p, s0 = pk
            if a.fused:
                qoq.w4a8_linear(X, p, s0, a.N, out=Y, workspace=ws, stream=s)
                continue
            if a.with_quant:
                qoq.quantize_activations_per_token(X, out=q, stream=s)
            qoq.w4a8_gemm(*q, p, s0, a.N, out=Y, workspace=ws, stream=s)

    with torch.cuda.stream(s):
        for _ in range(a.iters):
            run()
        s.synchronize()
        if a.time:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                run()
            for _ in range(3):
                g.replay()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(a.iters):
                g.replay()
            e1.record(s)
            s.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / (a.iters * a.layers)
            print(f"M={a.M} N={a.N} K={a.K}: {us:.2f} us/launch  "
                  f"{gemm_bytes(a.M, a.N, a.K) / us / 1e3:.0f} GB/s  {gemm_ops(a.M, a.N, a.K) / us / 1e6:.1f} TOPS")
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
