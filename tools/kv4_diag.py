import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import oracle, synth
import paper_2405_04532_b200 as qoq
from kv4_tol import kv4_tolerance
dev = torch.device("cuda:0")
T, Hq, Hkv, D, P = 70, 8, 2, 128, 64
Kx = synth.activations_fp16(T * Hkv, D, seed=2).reshape(T, Hkv, D)
Vx = synth.activations_fp16(T * Hkv, D, seed=3).reshape(T, Hkv, D)
bt = np.array([[1, 0]], np.int32)
pages = torch.zeros(2 * qoq.kv4_page_bytes(Hkv, D, P), dtype=torch.uint8, device=dev)
for t in range(T):
    slot = torch.tensor([bt[0, t // P] * P + t % P], dtype=torch.int32, device=dev)
    qoq.kv4_append(torch.from_numpy(np.ascontiguousarray(Kx[t:t + 1])).to(dev),
                   torch.from_numpy(np.ascontiguousarray(Vx[t:t + 1])).to(dev), slot, pages, P)
Q = synth.activations_fp16(Hq, D, seed=4).reshape(1, Hq, D)
O = qoq.kv4_decode_attention(torch.from_numpy(Q).to(dev), pages, torch.from_numpy(bt).to(dev),
                             torch.tensor([T], dtype=torch.int32, device=dev), Hkv, P)
torch.cuda.synchronize()
kq = oracle.kv4_quantize(Kx.reshape(-1, D)); vq = oracle.kv4_quantize(Vx.reshape(-1, D))
Kh = oracle.kv4_dequant(*kq).reshape(T, Hkv, D); Vh = oracle.kv4_dequant(*vq).reshape(T, Hkv, D)
o_ref = oracle.attention_f64(Q[0], Kh, Vh)
o = O.cpu().numpy()[0].astype(np.float64)
tol = kv4_tolerance(Q[0], Kh, Vh, o_ref)
err = np.abs(o - o_ref)
r = err / tol
i = np.unravel_index(np.argmax(r), r.shape)
print("max err/tol", r.max(), "at", i, "err", err[i], "tol", tol[i], "o", o[i], "ref", o_ref[i], "n bad", (r > 1).sum())
print("max |o-ref| rel", (err / (np.abs(o_ref) + 1e-30)).max(), "median tol", np.median(tol))
# per head softmax peakedness
q = Q[0].astype(np.float64)
for h in range(Hq):
    s = Kh[:, h // 4, :] @ q[h] / np.sqrt(D); p = np.exp(s - s.max()); p /= p.sum()
    print(h, "max score", s.max().round(1), "spread", (s.max() - s.min()).round(1), "p_max", p.max().round(4), "worst ratio head", r[h].max().round(2))
