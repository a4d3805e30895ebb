"""Per-CTA pipeline timeline of one W4A8 GEMM launch (debug entry qoq_debug_w4a8_gemm_trace).

Events (ns since the earliest CTA start): 0 start, 1 setup done, 2 producer past griddepcontrol.wait,
3 MMA first full stage, 4 MMA first expanded A, 5 MMA last commit, 6 epilogue acc ready,
7 partial reduced (pre-counter), 8 segment done, 9 tile finalized, 10 CTA end.
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# the stamps are compiled in only in the `trace` variant:
#   python paper_2405_04532_b200/build.py --variant=trace:-DQOQ_TRACING=1
os.environ.setdefault("QOQ_LIB_VARIANT", "trace")

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_04532_b200 as qoq  # noqa: E402
import synth  # noqa: E402

NAMES = ["start", "setup", "prod_pdl", "quant_rows", "handshake", "mma_done", "epi_acc", "epi_red", "seg_done",
         "finalized", "end", "mbar_init", "epi_pdl", "sync0", "epi_exit", "sync_end",
         "q_loaded", "q_scale", "q_stored", "q_row_done", "q_all_rows", "q_fence",
         "red_landed", "part_staged", "part_bar", "cl_acq", "epi_chunks", "epi_ld0", "epi_sts0", "epi_stg0", "epi_ld1", "epi_sts_done"]
EV = 32
IT = 148 * EV
CYC = IT + 64 * 8 + 16 * 8 * 2


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=64)
    ap.add_argument("--N", type=int, default=4096)
    ap.add_argument("--K", type=int, default=4096)
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--fused", action="store_true", help="trace qoq_w4a8_linear (fused quantization)")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    L = qoq.load()
    f = L.qoq_debug_w4a8_gemm_trace
    P, I, Z = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
    f.restype, f.argtypes = I, [P, P, P, P, P, I, I, I, P, P, Z, P, P]
    gen = torch.Generator(device=dev)
    packs = []
    for l in range(a.layers):
        gen.manual_seed(l)
        packs.append(qoq.quantize_weights(synth.device_weights_fp16(a.N, a.K, gen, dev)))
    X = synth.device_activations_fp16(a.M, a.K, gen, dev)
    qx, sx, tx = qoq.quantize_activations_per_token(X)
    Y = torch.empty(a.M, a.N, dtype=torch.float16, device=dev)
    wsb = qoq.gemm_workspace_bytes(a.M, a.N, a.K)
    ws = torch.zeros(max(wsb, 16), dtype=torch.uint8, device=dev)
    tr = torch.zeros(CYC + 148 * EV, dtype=torch.int64, device=dev)
    s = torch.cuda.current_stream()
    if a.fused:
        fl = L.qoq_debug_w4a8_linear_trace
        fl.restype, fl.argtypes = I, [P, I, I, I, P, P, P, P, Z, P, P]
        lwb = qoq.linear_workspace_bytes(a.M, a.N, a.K)
        lws = torch.zeros(lwb, dtype=torch.uint8, device=dev)
    for rep in range(3):
        for p, s0 in packs:
            tr.zero_()
            if a.fused:
                rc = fl(P(X.data_ptr()), a.M, a.N, a.K, P(p.data_ptr()), P(s0.data_ptr()), P(Y.data_ptr()),
                        P(lws.data_ptr()), lwb, P(tr.data_ptr()), P(s.cuda_stream))
                assert rc == 0, rc
                continue
            rc = f(P(qx.data_ptr()), P(sx.data_ptr()), P(tx.data_ptr()), P(p.data_ptr()), P(s0.data_ptr()),
                   a.M, a.N, a.K, P(Y.data_ptr()), P(ws.data_ptr()), wsb, P(tr.data_ptr()), P(s.cuda_stream))
            assert rc == 0, rc
    torch.cuda.synchronize()
    full = tr.cpu().numpy().astype(np.float64)
    t = full[:IT].reshape(-1, EV)
    its = full[IT:IT + 512].reshape(64, 8)
    mm = full[IT + 512:IT + 640].reshape(16, 8)
    dq = full[IT + 640:CYC].reshape(16, 8)
    cyc = full[CYC:].reshape(-1, EV)
    cyc = cyc[cyc[:, 0] > 0]
    crel = np.where(cyc > 0, cyc - cyc[:, :1], np.nan)
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    rel = np.where(t > 0, t - t0, np.nan)
    print(f"M={a.M} N={a.N} K={a.K}: {t.shape[0]} CTAs traced; kernel span {np.nanmax(rel[:, 10]) / 1e3:.2f} us")
    for e, n in enumerate(NAMES):
        col = rel[:, e]
        if np.all(np.isnan(col)):
            continue
        cc = crel[:, e]
        print(f"  {e:2d} {n:10s} min {np.nanmin(col) / 1e3:7.2f}  median {np.nanmedian(col) / 1e3:7.2f}  "
              f"max {np.nanmax(col) / 1e3:7.2f} us  (n={np.sum(~np.isnan(col))})   cycles from CTA start: "
              f"median {np.nanmedian(cc):8.0f} max {np.nanmax(cc):8.0f}")
    nz = its[its > 0]
    c0 = nz.min() if nz.size else 0
    print("  CTA 0 per step (SM cycles from first stamp): deq_wfull deq_regs deq_xready deq_st | mma_wait mma_go mma_iss | xprod")
    for i in range(64):
        row = its[i]
        if not np.any(row > 0):
            continue
        vals = ["   -   " if v == 0 else f"{int(v - c0):7d}" for v in row]
        print(f"   it{i:2d} " + " ".join(vals[:4]) + " | " + " ".join(vals[4:7]) + " | " + vals[7])
    print("  CTA 0 per-MMA issue stamps (cycles after mma_go of the step):")
    for i in range(16):
        if its[i, 5] > 0 and mm[i, 0] > 0:
            print(f"   it{i:2d} " + " ".join(f"{int(v - its[i, 5]):6d}" for v in mm[i] if v > 0))
    print("  CTA 0 per-warp dequant completion (cycles after the traced warp's xready) | mma_go - slowest")
    for i in range(16):
        if its[i, 2] > 0:
            done = [v for v in dq[i] if v > 0]
            if done:
                print(f"   it{i:2d} " + " ".join(f"{int(v - its[i, 2]):6d}" for v in done)
                      + f" | {int(its[i, 5] - max(done)):6d}")


if __name__ == "__main__":
    main()
