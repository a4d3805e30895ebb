"""Decode step through qoq_w4a8_linear_chain: Llama-3-8B, `layers` x (qkv, o, gate_up, down) at M tokens,
the whole step ONE launch (CUDA graph), vs the per-call path (quantizer + GEMM per linear, PDL).
Prints ms per step and GB/s of SURVEY §8(d) algorithmic bytes."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2405_04532_b200 as qoq  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, nargs="+", default=[64])
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--chained", action="store_true", help="X of o/gate_up... = previous Y where shapes allow")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    qoq.load()
    shapes = [(N, K) for _, N, K, _ in synth.fuse_gate_up(synth.LLAMA3_8B)]
    gen = torch.Generator(device=dev).manual_seed(0)
    packs = []
    for l in range(a.layers):
        row = []
        for N, K in shapes:
            row.append(qoq.quantize_weights(synth.device_weights_fp16(N, K, gen, dev)))
        packs.append(row)
    for M in a.M:
        X = {K: synth.device_activations_fp16(M, K, gen, dev) for _, K in shapes}
        Y = {N: torch.empty(M, N, dtype=torch.float16, device=dev) for N, _ in shapes}
        layers = []
        for l in range(a.layers):
            for (N, K), (p, s0) in zip(shapes, packs[l]):
                layers.append((X[K], p, s0, N, Y[N], K))
        ws = qoq.Workspace(dev)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            qoq.w4a8_linear_chain(layers, workspace=ws, stream=s)
            s.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                qoq.w4a8_linear_chain(layers, workspace=ws, stream=s)
            lws = qoq.Workspace(dev)
            for L in layers:
                qoq.w4a8_linear(L[0], L[1], L[2], L[3], out=torch.empty_like(L[4]), workspace=lws, stream=s)
            s.synchronize()
            g2 = torch.cuda.CUDAGraph()
            outs = [torch.empty_like(L[4]) for L in layers]
            with torch.cuda.graph(g2, stream=s):
                for L, o in zip(layers, outs):
                    qoq.w4a8_linear(L[0], L[1], L[2], L[3], out=o, workspace=lws, stream=s)
            res = {}
            for name, gr in (("chain", g), ("per_call", g2)):
                for _ in range(3):
                    gr.replay()
                s.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                for _ in range(a.reps):
                    gr.replay()
                e1.record(s)
                s.synchronize()
                res[name] = e0.elapsed_time(e1) / a.reps
        nbytes, _ = bench.step_work("llama3-8b", M, a.layers, 1)
        print(f"M={M:4d} layers={a.layers}: chain {res['chain']:.3f} ms ({nbytes / res['chain'] / 1e6:.0f} GB/s)  "
              f"per-call {res['per_call']:.3f} ms ({nbytes / res['per_call'] / 1e6:.0f} GB/s)", flush=True)


if __name__ == "__main__":
    main()
