"""Timeline of back-to-back W4A8 GEMM launches in a PDL chain (trace build; one trace buffer per launch, no
kernel between the launches, so the programmatic-dependent-launch overlap is what production sees).

  python tools/trace_chained.py --shapes 6144x4096,4096x4096,28672x4096,4096x14336 --M 64 --reps 4

For every launch after the first, times (us, %globaltimer, 256-ns ticks on B200) are relative to the END
of the previous launch (the latest CTA end): first CTA start, median setup done, median producer past
griddepcontrol.wait, median / max last MMA committed, median / max CTA end.
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("QOQ_LIB_VARIANT", "trace")

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_04532_b200 as qoq  # noqa: E402
import synth  # noqa: E402

EV = 32
IT = 148 * EV
CYC = IT + 64 * 8 + 16 * 8 * 2


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=64)
    ap.add_argument("--shapes", default="6144x4096,4096x4096,28672x4096,4096x14336")
    ap.add_argument("--reps", type=int, default=4)
    ap.add_argument("--with-quant", action="store_true",
                    help="launch the per-token quantizer before every GEMM, as the decode step does")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    L = qoq.load()
    f = L.qoq_debug_w4a8_gemm_trace
    P, I, Z = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
    f.restype, f.argtypes = I, [P, P, P, P, P, I, I, I, P, P, Z, P, P]
    gen = torch.Generator(device=dev)
    shapes = [tuple(int(v) for v in s.split("x")) for s in a.shapes.split(",")]
    work = []
    for rep in range(a.reps):
        for N, K in shapes:
            gen.manual_seed(len(work))
            p, s0 = qoq.quantize_weights(synth.device_weights_fp16(N, K, gen, dev))
            work.append((N, K, p, s0))
    Xf = {K: synth.device_activations_fp16(a.M, K, gen, dev) for K in {k for _, k in shapes}}
    Xs = {K: qoq.quantize_activations_per_token(Xf[K]) for K in Xf}
    Ys = {N: torch.empty(a.M, N, dtype=torch.float16, device=dev) for N in {n for n, _ in shapes}}
    wsb = max(qoq.gemm_workspace_bytes(a.M, N, K) for N, K in shapes)
    ws = torch.zeros(max(wsb, 16), dtype=torch.uint8, device=dev)
    trs = [torch.zeros(CYC + 148 * EV, dtype=torch.int64, device=dev) for _ in work]
    s = torch.cuda.Stream()

    def issue():
        for (N, K, p, s0), tr in zip(work, trs):
            qx, sx, tx = Xs[K]
            if a.with_quant:
                qoq.quantize_activations_per_token(Xf[K], out=Xs[K], stream=s)
            rc = f(P(qx.data_ptr()), P(sx.data_ptr()), P(tx.data_ptr()), P(p.data_ptr()), P(s0.data_ptr()),
                   a.M, N, K, P(Ys[N].data_ptr()), P(ws.data_ptr()), wsb, P(tr.data_ptr()), P(s.cuda_stream))
            assert rc == 0, rc

    # the launch sequence as ONE CUDA graph (as the bench step): host enqueue cost out of the timeline
    with torch.cuda.stream(s):
        issue()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        issue()
    for _ in range(2):
        for t in trs:
            t.zero_()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
    prev_end = None
    print(f"M={a.M}: us relative to the previous launch's last CTA end "
          "(start_min | setup_med | pdl_med | mma_med mma_max | end_med end_max | span)")
    for (N, K, _, _), tr in zip(work, trs):
        t = tr.cpu().numpy()[:IT].reshape(-1, EV).astype(np.float64)
        t = t[t[:, 0] > 0]
        if prev_end is None:
            prev_end = t[:, 10].max()
            continue
        r = (t - prev_end) / 1e3
        r[t == 0] = np.nan
        print(f"  {N:6d}x{K:<6d} G={t.shape[0]:3d}: start {np.nanmin(r[:, 0]):6.2f} | setup {np.nanmedian(r[:, 1]):6.2f} | "
              f"pdl {np.nanmedian(r[:, 2]):6.2f} | mma {np.nanmedian(r[:, 5]):6.2f} {np.nanmax(r[:, 5]):6.2f} | "
              f"end {np.nanmedian(r[:, 10]):6.2f} {np.nanmax(r[:, 10]):6.2f} | span {(t[:, 10].max() - t[:, 0].min()) / 1e3:6.2f}")
        prev_end = t[:, 10].max()


if __name__ == "__main__":
    main()
