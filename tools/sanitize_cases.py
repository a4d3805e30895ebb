"""Small invocations of every kernel family for compute-sanitizer (tools/sanitize.sh): the per-call GEMM
in each planner mode (0 whole tiles, 1 stream-K, 2 cluster split-K), the CTA-pair variant, the fused
linear (grid handshake), per-channel W4A8, the quantizers (plain, RMSNorm, SiLU·mul), the KV4 cache +
decode attention, and the persistent decode chain. Each case checks its result against the CUDA path's
own reference call where one exists (the parity suites do the oracle comparisons)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2405_04532_b200 as qoq  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")


def gemm(mode=None, cg=None, M=16, N=256, K=512):
    if mode is not None:
        os.environ["QOQ_FORCE_MODE"] = str(mode)
    if cg is not None:
        os.environ["QOQ_FORCE_CG"] = str(cg)
    try:
        gen = torch.Generator(device=dev).manual_seed(1)
        p, s0 = qoq.quantize_weights(synth.device_weights_fp16(N, K, gen, dev))
        qx, sx, tx = qoq.quantize_activations_per_token(synth.device_activations_fp16(M, K, gen, dev))
        ws = qoq.Workspace(dev)
        y = qoq.w4a8_gemm(qx, sx, tx, p, s0, N, workspace=ws)
        a = qoq.w4a8_gemm_i32(qx, None, p, N, workspace=ws)
        torch.cuda.synchronize()
        assert torch.isfinite(y.float()).all() and a.abs().sum() > 0
    finally:
        os.environ.pop("QOQ_FORCE_MODE", None)
        os.environ.pop("QOQ_FORCE_CG", None)


def fused_linear(M=16, N=256, K=512):
    os.environ["QOQ_LINEAR_FUSED"] = "1"
    try:
        gen = torch.Generator(device=dev).manual_seed(2)
        p, s0 = qoq.quantize_weights(synth.device_weights_fp16(N, K, gen, dev))
        X = synth.device_activations_fp16(M, K, gen, dev)
        y1 = qoq.w4a8_linear(X, p, s0, N)
        os.environ.pop("QOQ_LINEAR_FUSED")
        y2 = qoq.w4a8_linear(X, p, s0, N)
        torch.cuda.synchronize()
        assert torch.equal(y1, y2)
    finally:
        os.environ.pop("QOQ_LINEAR_FUSED", None)


def per_channel(M=16, N=256, K=512):
    gen = torch.Generator(device=dev).manual_seed(3)
    p, sw, zw = qoq.pc_quantize_weights(synth.device_weights_fp16(N, K, gen, dev))
    qx, sx, tx = qoq.quantize_activations_per_token(synth.device_activations_fp16(M, K, gen, dev))
    y = qoq.pc_w4a8_gemm(qx, sx, tx, p, sw, zw, N)
    torch.cuda.synchronize()
    assert torch.isfinite(y.float()).all()


def quantizers(M=8, K=512):
    gen = torch.Generator(device=dev).manual_seed(4)
    X = synth.device_activations_fp16(M, K, gen, dev)
    g = (1 + 0.1 * torch.randn(K, generator=gen, device=dev)).half()
    qoq.rmsnorm_quantize(X, g, 1e-5)
    qoq.silu_mul_quantize(torch.randn(M, 2 * K, generator=gen, device=dev).half())
    torch.cuda.synchronize()


def kv4(B=2, T=70, H=8, H_kv=2, D=128, P=64):
    gen = torch.Generator(device=dev).manual_seed(5)
    npg = (T + P - 1) // P
    pages = torch.zeros(B * npg * qoq.kv4_page_bytes(H_kv, D, P), dtype=torch.uint8, device=dev)
    bt = torch.arange(B * npg, dtype=torch.int32, device=dev).view(B, npg)
    for t in range(T):
        slots = (bt[:, t // P] * P + t % P).contiguous()
        qoq.kv4_append(torch.randn(B, H_kv, D, generator=gen, device=dev).half(),
                       torch.randn(B, H_kv, D, generator=gen, device=dev).half(), slots, pages, P)
    O = qoq.kv4_decode_attention(torch.randn(B, H, D, generator=gen, device=dev).half(), pages, bt,
                                 torch.tensor([T, T - 7], dtype=torch.int32, device=dev), H_kv, P)
    torch.cuda.synchronize()
    assert torch.isfinite(O.float()).all()


def chain(M=16):
    gen = torch.Generator(device=dev).manual_seed(6)
    shapes = [(256, 256), (512, 256), (256, 512)]
    layers, prev = [], None
    for N, K in shapes:
        p, s0 = qoq.quantize_weights(synth.device_weights_fp16(N, K, gen, dev))
        X = prev if prev is not None and prev.shape[1] == K else synth.device_activations_fp16(M, K, gen, dev)
        Y = torch.empty(M, N, dtype=torch.float16, device=dev)
        layers.append((X, p, s0, N, Y, K))
        prev = Y
    qoq.w4a8_linear_chain(layers)
    torch.cuda.synchronize()
    remap = {}
    for X, p, s0, N, Y, K in layers:
        r = qoq.w4a8_linear(remap.get(X.data_ptr(), X), p, s0, N)
        remap[Y.data_ptr()] = r
        assert torch.equal(r, Y)


def tp_fused(M=16, N=256, K=512):
    """NEXT-3: the fused TP reduction at world 1 (push + flag-in-data words + rank-order reduce, all local)
    equals the plain GEMM, over both buffer parities."""
    gen = torch.Generator(device=dev).manual_seed(3)
    p, s0 = qoq.quantize_weights(synth.device_weights_fp16(N, K, gen, dev))
    qx, sx, tx = qoq.quantize_activations_per_token(synth.device_activations_fp16(M, K, gen, dev))
    ref = qoq.w4a8_gemm(qx, sx, tx, p, s0, N)
    comm = qoq.TpComm.local(M, N, dev)
    for _ in range(2):
        y = qoq.w4a8_gemm_allreduce(qx, sx, tx, p, s0, N, comm)
        torch.cuda.synchronize()
        assert torch.equal(y, ref) and comm.status() == 0


CASES = {"gemm_mode0": lambda: gemm(mode=0), "gemm_mode1": lambda: gemm(mode=1, M=64, N=256, K=1024),
         "gemm_mode2": lambda: gemm(mode=2, M=16, N=256, K=1024), "gemm_cg2": lambda: gemm(cg=2, M=64, N=256, K=512),
         "gemm_prefill": lambda: gemm(M=300, N=256, K=256), "fused_linear": fused_linear, "per_channel": per_channel,
         "quantizers": quantizers, "kv4": kv4, "chain": chain, "tp_fused": tp_fused}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="all")
    a = ap.parse_args()
    qoq.load()
    for name, fn in CASES.items():
        if a.case in ("all", name):
            fn()
            print(f"case {name}: ok", flush=True)
