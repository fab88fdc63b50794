"""BASELINE config 3 on ONE B200: a stack of L MEFT adapter layers (d=4096, M=65,536, 256 experts, K=128) with
all tables and Adam state resident in HBM, T tokens per step (16,384 in the config). One step = the fused layer
step of every layer in turn. With fp32 Adam moments (MIXED, 7.5 GB per layer) 32 layers need ~240 GB, so 22 fit
one GPU; with bf16 moments (COMPACT, 5.4 GB per layer) all 32 do.

  python tools/stack_bench.py [layers=20] [tokens=16384] [steps=3] [mixed|compact] [sync|enqueue|graph]

sync (default): each layer step reads |S| back once mid-step (meft_layer_step's host sync); enqueue: host sync off
(meft_ctx_set_host_sync), the layers enqueue back to back with no read-back; graph: the whole L-layer step captured
once into a CUDA graph (meft_graph_*) and replayed.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_04984_b200 import meft as G  # noqa: E402


def main():
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    prec = sys.argv[4] if len(sys.argv) > 4 else "mixed"
    mode = sys.argv[5] if len(sys.argv) > 5 else "sync"
    assert mode in ("sync", "enqueue", "graph"), mode
    d, M, N, K, kk = 4096, 65536, 256, 128, 4
    stream = torch.cuda.Stream() if mode == "graph" else torch.cuda.current_stream()  # default stream: no capture
    torch.cuda.set_stream(stream)
    ctx = G.Context(0, stream=stream)
    ctx.set_host_sync(mode == "sync")
    st = G.Store(ctx, L, d, M, N, G.STORE_COMPACT if prec == "compact" else G.STORE_MIXED)
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
    out = torch.empty((T, d), device="cuda")  # per-layer results (overwritten layer by layer, as a trainer would consume)
    gh = torch.empty((T, d), device="cuda")

    def stack_step():
        for layer in range(L):
            st.layer_step(layer, h, g, kk, K, 1e-4, out=out, grad_h=gh, want_info=(mode == "sync"))

    stack_step()  # warm-up: every layer once (allocates every scratch buffer)
    torch.cuda.synchronize()
    graph = None
    if mode == "graph":
        with ctx.graph() as graph:
            stack_step()
        graph.replay()  # first replay uploads the graph
        torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        if graph is not None:
            graph.replay()
        else:
            stack_step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    per_layer = ms / L
    free, total = torch.cuda.mem_get_info()
    print(json.dumps({"layers_resident": L, "precision": prec, "mode": mode, "tokens_per_step": T, "ms_per_step": ms, "ms_per_layer": per_layer,
                      "tokens_per_s": T / ms * 1e3, "layer_tokens_per_s": T * L / ms * 1e3,
                      "projected_32_layer_ms": 32 * per_layer, "projected_32_layer_tokens_per_s": T / (32 * per_layer) * 1e3,
                      "hbm_used_gb": (total - free) / 1e9}))


if __name__ == "__main__":
    main()
