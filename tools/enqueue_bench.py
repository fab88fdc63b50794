"""Host-sync A/B of the fused layer step: the same L-layer stack stepped with host sync on (each layer step reads |S|
back mid-step), off (enqueue-only: meft_ctx_set_host_sync(ctx, 0)), and as one captured CUDA graph, interleaved
`reps` times on one GPU; prints one JSON line per (mode, rep) and a median summary.

  python tools/enqueue_bench.py cfg1|cfg2 [layers=4] [steps=20] [reps=3]

cfg1 = BASELINE configs[0] (d=512, M=4,096, 64 experts, K=32, T=256): launch- and sync-bound;
cfg2 = configs[1] (d=4096, M=65,536, 256 experts, K=128, T=8,192): GEMM-bound.
"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_04984_b200 import meft as G  # noqa: E402

SHAPES = {"cfg1": (512, 4096, 64, 32, 4, 256), "cfg2": (4096, 65536, 256, 128, 4, 8192)}


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
    L = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
    d, M, N, K, kk, T = SHAPES[cfg]
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = G.Context(0, stream=stream)
    st = G.Store(ctx, L, d, M, N, G.STORE_MIXED)
    b = 1.0 / d ** 0.5
    gen = torch.Generator(device="cuda").manual_seed(1)
    with torch.no_grad():
        for layer in range(L):
            for name in ("w_a", "w_b", "w_g"):
                w = st.tensor(layer, name)
                w.uniform_(-b, b, generator=gen)
                st.tensor(layer, name + "_compute").copy_(w.to(torch.bfloat16))
    h = (torch.rand((T, d), generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16)
    g = (torch.rand((T, d), generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16)
    out = torch.empty((T, d), device="cuda")
    gh = torch.empty((T, d), device="cuda")

    def stack_step(info):
        for layer in range(L):
            st.layer_step(layer, h, g, kk, K, 1e-4, out=out, grad_h=gh, want_info=info)

    ctx.set_host_sync(False)
    stack_step(False)  # warm-up (allocations), then capture the enqueue-only stack step
    torch.cuda.synchronize()
    with ctx.graph() as graph:
        stack_step(False)
    graph.replay()
    torch.cuda.synchronize()

    def run(mode):
        ctx.set_host_sync(mode == "sync")
        stack_step(mode == "sync")  # one untimed step in this mode
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            if mode == "graph":
                graph.replay()
            else:
                stack_step(mode == "sync")
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / steps

    res = {m: [] for m in ("sync", "enqueue", "graph")}
    for rep in range(reps):
        for mode in res:
            ms = run(mode)
            res[mode].append(ms)
            print(json.dumps({"config": cfg, "layers": L, "tokens": T, "mode": mode, "rep": rep,
                              "ms_per_step": ms, "ms_per_layer": ms / L, "tokens_per_s": T / ms * 1e3}))
    med = {m: statistics.median(v) for m, v in res.items()}
    print(json.dumps({"config": cfg, "layers": L, "steps": steps, "reps": reps,
                      "median_ms_per_layer": {m: v / L for m, v in med.items()},
                      "speedup_vs_sync": {m: med["sync"] / v for m, v in med.items()}}))
    graph.close()


if __name__ == "__main__":
    main()
