"""Prefill GEMM TOPS per Llama-3-8B projection and M under the planner's choice vs forced decompositions
(QOQ_FORCE_MODE / QOQ_BN_BIG), 4 rotating layers of weights, CUDA graph per projection."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2405_04532_b200 as qoq  # noqa: E402
import synth  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    qoq.load()
    shapes = [(n, N, K) for n, N, K, _ in synth.fuse_gate_up(synth.LLAMA3_8B)]
    gen = torch.Generator(device=dev).manual_seed(0)
    L = 4
    packs = {n: [qoq.quantize_weights(synth.device_weights_fp16(N, K, gen, dev)) for _ in range(L)] for n, N, K in shapes}
    s = torch.cuda.Stream()
    for M in (1024, 2048, 4096):
        acts = {K: qoq.quantize_activations_per_token(synth.device_activations_fp16(M, K, gen, dev)) for K in {k for _, _, k in shapes}}
        for label, env in (("auto", {}), ("mode1", {"QOQ_FORCE_MODE": "1"}), ("bn192", {"QOQ_BN_BIG": "192"}),
                           ("bn256", {"QOQ_BN_BIG": "256"})):
            for k in ("QOQ_FORCE_MODE", "QOQ_BN_BIG"):
                os.environ.pop(k, None)
            os.environ.update(env)
            row = []
            for n, N, K in shapes:
                qx, sx, tx = acts[K]
                Y = torch.empty(M, N, dtype=torch.float16, device=dev)
                ws = qoq.Workspace(dev)
                with torch.cuda.stream(s):
                    for p, s0 in packs[n]:
                        qoq.w4a8_gemm(qx, sx, tx, p, s0, N, out=Y, workspace=ws, stream=s)
                    s.synchronize()
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=s):
                        for p, s0 in packs[n]:
                            qoq.w4a8_gemm(qx, sx, tx, p, s0, N, out=Y, workspace=ws, stream=s)
                    g.replay()
                    s.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(s)
                    for _ in range(5):
                        g.replay()
                    e1.record(s)
                    s.synchronize()
                ms = e0.elapsed_time(e1) / 5 / L
                row.append(f"{n} {2 * M * N * K / ms / 1e9:6.0f}")
            print(f"M={M:5d} {label:6s}: " + "  ".join(row), flush=True)
    for k in ("QOQ_FORCE_MODE", "QOQ_BN_BIG"):
        os.environ.pop(k, None)


if __name__ == "__main__":
    main()
