"""Repeat one W4A8 INT32 GEMM against the oracle through a given library file (raw ctypes, no ABI
check) — for bisecting a parity failure across builds.

  QOQ_FORCE_MODE=1 python tools/repro_gemm.py --lib paper_2405_04532_b200/libqoq_b200.so --M 5 --N 2560 --K 1408
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", required=True)
    ap.add_argument("--M", type=int, default=5)
    ap.add_argument("--N", type=int, default=2560)
    ap.add_argument("--K", type=int, default=1408)
    ap.add_argument("--seed", type=int, default=-1)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--no-tx", action="store_true")
    a = ap.parse_args()
    L = ctypes.CDLL(os.path.abspath(a.lib))
    P, I, Z = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
    L.qoq_gemm_workspace_bytes.restype, L.qoq_gemm_workspace_bytes.argtypes = Z, [I, I, I]
    L.qoq_w4a8_gemm_i32.restype = I
    L.qoq_w4a8_gemm_i32.argtypes = [P, P, P, I, I, I, I, P, I, P, Z, P]
    M, N, K = a.M, a.N, a.K
    seed = a.seed if a.seed >= 0 else M + K
    W = synth.weights_fp16(N, K, seed=seed)
    X = synth.activations_fp16(M, K, seed=seed)
    p_ref, s0_ref = oracle.quantize_weights(W)
    qx_ref, sx_ref, tx_ref = oracle.quantize_activations(X)
    acc_ref = oracle.acc_from_packed(qx_ref, p_ref, N, K)
    dev = torch.device("cuda:0")
    qx = torch.from_numpy(qx_ref).to(dev)
    tx = torch.from_numpy(tx_ref).to(dev)
    pk = torch.from_numpy(p_ref).to(dev)
    wsb = L.qoq_gemm_workspace_bytes(M, N, K)
    ws = torch.zeros(max(wsb, 16), dtype=torch.uint8, device=dev)
    acc = torch.empty(M, N, dtype=torch.int32, device=dev)
    bad_runs = 0
    for r in range(a.reps):
        acc.fill_(0x7F7F7F7F)
        rc = L.qoq_w4a8_gemm_i32(P(qx.data_ptr()), None if a.no_tx else P(tx.data_ptr()), P(pk.data_ptr()), M, N, K,
                                 128, P(acc.data_ptr()), N, P(ws.data_ptr()), wsb, None)
        torch.cuda.synchronize()
        assert rc == 0, rc
        d = acc.cpu().numpy() != acc_ref
        if d.any():
            bad_runs += 1
            rows, cols = np.nonzero(d)
            print(f"rep {r}: {d.sum()} differ; rows {sorted(set(rows.tolist()))} cols {cols.min()}..{cols.max()} "
                  f"tiles {sorted(set((cols // 128).tolist()))[:12]}; ws nonzero {int(ws.count_nonzero())}")
    print(f"{os.path.basename(a.lib)} mode={os.environ.get('QOQ_FORCE_MODE', 'auto')} M={M} N={N} K={K}: "
          f"{bad_runs}/{a.reps} runs wrong")


if __name__ == "__main__":
    main()
