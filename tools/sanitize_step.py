"""compute-sanitizer target (profiles/r2_sanitizer_*.txt): small but complete runs of the hot path --
two fused layer steps at BASELINE config 1 (MIXED store: certified selection, tcgen05 FFN GEMMs, Adam epilogue),
one step on a COMPACT store, and two steps of the C-ABI expert-sharded layer at world 1 over the library's own
NCCL communicator.
  compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_step.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_04984_b200 import meft as G  # noqa: E402
from paper_2406_04984_b200 import sharded as SH  # noqa: E402


def store(ctx, prec, d, M, N):
    st = G.Store(ctx, 1, d, M, N, prec)
    b = 1.0 / d ** 0.5
    st.upload(0, "w_a", G.reference_uniform(1, 0x5000, (d, M), -b, b, bf16=True))
    st.upload(0, "w_g", G.reference_uniform(1, 0x5001, (N, d), -b, b, bf16=True))
    st.upload(0, "w_b", G.reference_uniform(1, 0x7001, (M, d), -b, b, bf16=True))
    return st


def main():
    d, M, N, K, kk, T = 512, 4096, 64, 32, 4, 256
    ctx = G.Context(0)
    h = torch.from_numpy(G.reference_uniform(1, 0x7002, (T, d), -1, 1, bf16=True)).cuda().bfloat16()
    g = torch.from_numpy(G.reference_uniform(1, 0x7003, (T, d), -1, 1, bf16=True)).cuda().bfloat16()
    out = torch.empty((T, d), device="cuda")
    gh = torch.empty_like(out)
    st = store(ctx, G.STORE_MIXED, d, M, N)
    for _ in range(2):
        r = st.layer_step(0, h, g, kk, K, 1e-3, out=out, grad_h=gh, want_selection=True)
    torch.cuda.synchronize()
    print("mixed layer steps ok, |S| =", r["union_size"], flush=True)
    cst = store(ctx, G.STORE_COMPACT, d, M, N)
    cst.layer_step(0, h, g, kk, K, 1e-3, out=out, grad_h=gh)
    torch.cuda.synchronize()
    print("compact layer step ok", flush=True)
    sh = store(ctx, G.STORE_MIXED, d, M, N)
    layer = SH.CShardedLayer(ctx, sh, sh.tensor(0, "w_g_compute").clone())
    for _ in range(2):
        res = layer.step(h, g, kk, K, 1e-3)
    torch.cuda.synchronize()
    layer.close()
    print("sharded (C ABI, NCCL world 1) steps ok, |S| =", res["union_size"], flush=True)


if __name__ == "__main__":
    main()
