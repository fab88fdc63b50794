"""Developer harness: the HBM-bound reference-API kernels alone at cfg2 (for ncu captures): fetch (row gather of
the selected key/value rows), scatter_grads (row scatter-add into the staging tables) and sparse_adam_update
(staged pairs), over S = a random half of the 65,536 pairs (ascending, unique: the reference's union).
   python tools/profile_hbm.py [iters]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_04984_b200 import meft as G  # noqa: E402


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    d, M, N = 4096, 65536, 256
    ctx = G.Context(0)
    st = G.Store(ctx, 1, d, M, N, G.STORE_MIXED)
    st.init_reference(seed=1)
    gen = torch.Generator(device="cuda").manual_seed(3)
    S = torch.sort(torch.randperm(M, generator=gen, device="cuda")[: M // 2]).values.to(torch.int32).contiguous()
    s = S.numel()
    gk = torch.randn((s, d), generator=gen, device="cuda") * 1e-3
    gv = torch.randn((s, d), generator=gen, device="cuda") * 1e-3
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    for i in range(iters):
        ev[0].record(torch.cuda.current_stream())
        ks, vs = st.fetch(0, S)
        ev[1].record(torch.cuda.current_stream())
        st.scatter_grads(0, S, gk, gv)
        ev[2].record(torch.cuda.current_stream())
        st.sparse_adam_update(0, 1e-4)
        ev[3].record(torch.cuda.current_stream())
        torch.cuda.synchronize()
    f, sc, a = (ev[i].elapsed_time(ev[i + 1]) for i in range(3))
    gb = lambda b, ms: b / (ms * 1e-3) / 1e9  # noqa: E731
    print(f"|S|={s}: fetch {f:.3f} ms ({gb(2 * s * d * 2 * 2, f):.0f} GB/s), scatter {sc:.3f} ms "
          f"({gb(2 * s * d * (4 + 4 + 4), sc):.0f} GB/s), adam {a:.3f} ms ({gb(2 * s * d * 34, a):.0f} GB/s)")


if __name__ == "__main__":
    main()
