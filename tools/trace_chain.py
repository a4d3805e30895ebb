"""Timeline of one qoq_w4a8_linear_chain launch (debug entry qoq_debug_w4a8_linear_chain_trace, `trace`
library variant: python paper_2405_04532_b200/build.py --variant=trace:-DQOQ_TRACING=1).
Per linear j, over CTAs (us from the earliest stamp): 0 quantization start (Y_{j-1} complete seen),
1 quantization released, 2 q_x acquired by the activation producer, 3 first MMA, 4 last MMA commit,
5 epilogue done, 6 first weights in SMEM, 7 first weight copy issued."""
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

EV = ["q_start", "q_rel", "x_acq", "mma0", "mma_end", "epi_end", "w_in", "w_iss", "q_staged", "q_scale", "q_stored",
      "q_prerel", "acc0", "announce", "landed0", "fin_done", "p_staged", "p_issued", "p_stored", "f_loaded",
      "f_summed", "x_iss0", "m_afull", "m_xfull", "m_issued", "q_ready"] + [f"e{i}" for i in range(26, 32)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=64)
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--same-weights", action="store_true", help="every layer reuses layer 0's weights (L2-resident)")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    L = qoq.load()
    f = L.qoq_debug_w4a8_linear_chain_trace
    P = ctypes.c_void_p
    f.restype, f.argtypes = ctypes.c_int, [ctypes.c_int, ctypes.c_int, P, P, ctypes.c_size_t, P, P]
    shapes = [(N, K) for _, N, K, _ in synth.fuse_gate_up(synth.LLAMA3_8B)]
    gen = torch.Generator(device=dev).manual_seed(0)
    layers = []
    X = {K: synth.device_activations_fp16(a.M, K, gen, dev) for _, K in shapes}
    Y = {N: torch.empty(a.M, N, dtype=torch.float16, device=dev) for N, _ in shapes}
    packs = {}
    for l in range(a.layers):
        for N, K in shapes:
            if not a.same_weights or (N, K) not in packs:
                packs[N, K] = qoq.quantize_weights(synth.device_weights_fp16(N, K, gen, dev))
            p, s0 = packs[N, K]
            layers.append((X[K], p, s0, N, Y[N], K))
    M, arr = qoq.chain_descs(layers)
    n = len(arr)
    nb = L.qoq_linear_chain_workspace_bytes(M, n, arr)
    ws = torch.zeros(nb, dtype=torch.uint8, device=dev)
    G = torch.cuda.get_device_properties(dev).multi_processor_count
    tr = torch.zeros(2 * n * G * 32, dtype=torch.int64, device=dev)
    s = torch.cuda.current_stream()
    for rep in range(4):
        tr.zero_()
        rc = f(M, n, arr, P(ws.data_ptr()), nb, P(tr.data_ptr()), P(s.cuda_stream))
        assert rc == 0, rc
    torch.cuda.synchronize()
    full = tr.cpu().numpy().astype(np.float64)
    t = full[:n * G * 32].reshape(n, G, 32)
    cyc = full[n * G * 32:].reshape(n, G, 32)
    t0 = t[t > 0].min()
    rel = np.where(t > 0, (t - t0) / 1e3, np.nan)
    span = np.nanmax(rel)
    print(f"M={M} linears={n} ({a.layers} Llama-3-8B layers): kernel span {span:.2f} us "
          f"({span / a.layers:.2f} us per layer)")
    print("  j   shape         " + " ".join(f"{e:>17s}" for e in EV[:8]))
    names = ["qkv", "o", "gate_up", "down"]
    for j in range(n):
        cells = []
        for e in range(26):
            c = rel[j, :, e]
            if np.all(np.isnan(c)):
                cells.append(f"{'-':>17s}")
            else:
                cells.append(f"{np.nanmedian(c):8.2f}/{np.nanmax(c):8.2f}")
        print(f"  {j:2d} {names[j % 4]:8s} " + " ".join(cells[:8]))
        print(f"  {'':11s} " + " ".join(f"{e[:8]:>8s}:{c.strip()}" for e, c in zip(EV[8:16], cells[8:16])))
        print(f"  {'':11s} " + " ".join(f"{e[:8]:>8s}:{c.strip()}" for e, c in zip(EV[16:26], cells[16:26])))
    print("  (each cell: median/max over CTAs, us)")
    # boundary breakdown: previous linear's last epilogue -> quantization -> activations -> first MMA
    print("  boundary j-1 -> j (us): epi_end(j-1,max) -> q_start(j,min) -> q_rel(j,max) -> x_acq(j,median) "
          "-> mma0(j,median); mma_end(j,max) - mma0(j,median)")
    for j in range(1, n):
        e5 = np.nanmax(rel[j - 1, :, 5])
        q0 = np.nanmin(rel[j, :, 0])
        q1 = np.nanmax(rel[j, :, 1])
        x2 = np.nanmedian(rel[j, :, 2])
        m3 = np.nanmedian(rel[j, :, 3])
        m4 = np.nanmax(rel[j, :, 4])
        print(f"  {j:2d} {names[j % 4]:8s} {e5:8.2f} -> {q0 - e5:+6.2f} -> {q1 - q0:+6.2f} -> {x2 - q1:+6.2f} -> "
              f"{m3 - x2:+6.2f};  main {m4 - m3:6.2f}; epi tail {np.nanmax(rel[j, :, 5]) - m4:6.2f}")
    cycles_report(cyc, n, names)


def cycles_report(cyc, n, names):
    """intra-CTA phase lengths in SM cycles (median over CTAs that recorded both stamps)"""
    pairs = [("q_start", "q_staged"), ("q_staged", "q_scale"), ("q_scale", "q_stored"), ("q_stored", "q_prerel"),
             ("q_prerel", "q_rel"), ("x_acq", "x_iss0"), ("x_iss0", "m_xfull"), ("m_xfull", "m_issued"),
             ("x_acq", "mma_end"), ("acc0", "p_staged"), ("p_staged", "p_issued"), ("p_issued", "p_stored"),
             ("p_stored", "announce"), ("announce", "landed0"), ("landed0", "f_loaded"), ("f_loaded", "f_summed"),
             ("f_summed", "fin_done"), ("fin_done", "epi_end")]
    print("  intra-CTA phases, SM cycles (median / max over CTAs):")
    for k, (a, b) in enumerate(pairs):
        print(f"   [{k:2d}] {a} -> {b}")
    print("  j   shape    " + " ".join(f"[{k:2d}]{'':10s}" for k in range(len(pairs))))
    for j in range(n):
        cells = []
        for a, b in pairs:
            x, y = cyc[j, :, EV.index(a)], cyc[j, :, EV.index(b)]
            ok = (x > 0) & (y > 0)
            d = (y - x)[ok]
            cells.append(f"{np.median(d):7.0f}/{d.max():7.0f}" if d.size else f"{'-':>15s}")
        print(f"  {j:2d} {names[j % 4]:8s} " + " ".join(cells))


if __name__ == "__main__":
    main()
