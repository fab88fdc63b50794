"""Developer harness: Key-Experts selection alone (for ncu launch lists / captures), cfg2 shape by default.
   python tools/profile_select.py [iters] [exact|certified] [M:N:K]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_04984_b200 import meft as G  # noqa: E402


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    exact = len(sys.argv) > 2 and sys.argv[2] == "exact"
    d, M, N, K, kk, T = 4096, 65536, 256, 128, 4, 8192
    if len(sys.argv) > 3:
        M, N, K = (int(x) for x in sys.argv[3].split(":"))
    gen = torch.Generator(device="cuda").manual_seed(5)
    rnd = lambda shape, s: ((torch.rand(shape, generator=gen, device="cuda") * 2 - 1) * s).to(torch.bfloat16)  # noqa
    h, keys, w_g = rnd((T, d), 1.0), rnd((M, d), 1 / 64), rnd((N, d), 1 / 64)
    ctx = G.Context(0)
    ctx.set_selection(exact)
    for _ in range(2):
        G.ke_select(ctx, h, w_g, keys, kk, K)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        sel = G.ke_select(ctx, h, w_g, keys, kk, K)
    e1.record()
    torch.cuda.synchronize()
    print(f"M={M} N={N} K={K} ke_select {'exact' if exact else 'certified'}: {e0.elapsed_time(e1) / iters:.3f} ms/call, |S|={sel.unioned.numel()}")


if __name__ == "__main__":
    main()
