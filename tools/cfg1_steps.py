"""Developer harness: N fused layer steps at BASELINE cfg1 (d=512, M=4096, 64 experts, K=32, T=256), for ncu launch
lists of the launch-bound small configuration.   python tools/cfg1_steps.py [steps] [sync|enqueue]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_04984_b200 import meft as G  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    mode = sys.argv[2] if len(sys.argv) > 2 else "sync"
    d, M, N, K, kk, T = 512, 4096, 64, 32, 4, 256
    ctx = G.Context(0)
    ctx.set_host_sync(mode == "sync")
    st = G.Store(ctx, 1, d, M, N, G.STORE_MIXED)
    b = 1.0 / d ** 0.5
    st.upload(0, "w_a", G.reference_uniform(1, 0x5000, (d, M), -b, b, bf16=True))
    st.upload(0, "w_g", G.reference_uniform(1, 0x5001, (N, d), -b, b, bf16=True))
    st.upload(0, "w_b", G.reference_uniform(1, 0x7001, (M, d), -b, b, bf16=True))
    h = torch.from_numpy(G.reference_uniform(1, 0x7002, (T, d), -1, 1, bf16=True)).cuda().bfloat16()
    g = torch.from_numpy(G.reference_uniform(1, 0x7003, (T, d), -1, 1, bf16=True)).cuda().bfloat16()
    out = torch.empty((T, d), device="cuda")
    gh = torch.empty_like(out)
    for _ in range(steps):
        st.layer_step(0, h, g, kk, K, 1e-4, out=out, grad_h=gh, want_info=(mode == "sync"))
    torch.cuda.synchronize()
    print("done")


if __name__ == "__main__":
    main()
