"""Run qoq_kv4_decode_attention once at the bench size (for ncu captures).

  python tools/prof_kv4.py [--B 64 --T 1024]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2405_04532_b200 as qoq  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--B", type=int, default=64)
    ap.add_argument("--T", type=int, default=1024)
    a = ap.parse_args()
    H, H_kv, D, P = 32, 8, 128, 64
    dev = torch.device("cuda:0")
    qoq.load()
    npg = a.T // P
    pages = torch.randint(0, 256, (a.B * npg * qoq.kv4_page_bytes(H_kv, D, P),), dtype=torch.uint8, device=dev)
    pv = pages.view(a.B * npg, H_kv, P * (D + 8))
    par = pv[:, :, P * D:].contiguous().view(torch.float16)
    par.copy_(torch.rand_like(par) * 0.01)                 # finite fp16 scale/zero pairs
    pv[:, :, P * D:] = par.view(torch.uint8).view(a.B * npg, H_kv, P * 8)
    bt = torch.randperm(a.B * npg, device=dev).to(torch.int32).view(a.B, npg)
    lens = torch.full((a.B,), a.T, dtype=torch.int32, device=dev)
    Q = torch.randn(a.B, H, D, device=dev).half()
    for _ in range(2):
        qoq.kv4_decode_attention(Q, pages, bt, lens, H_kv, P)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
