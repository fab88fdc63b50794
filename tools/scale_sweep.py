"""Scale sweep on ONE B200 (BASELINE.json configs 4-5 at a single GPU): fused layer step throughput over neuron
count M and per-token budget K. Tables are initialised on the device (uniform +-1/sqrt(d), bf16 compute copies),
inputs uniform(-1, 1); each point prints one JSON line. Points that do not fit HBM report the error.

  python tools/scale_sweep.py [T] M:N:K [M:N:K ...]      e.g.  8192 65536:256:128 1048576:1024:128
With MEFT_SWEEP_CPU=1 every point whose fp64 reference store fits host RAM (M <= 65536 here) is also timed on the
unmodified reference CPU implementation (oracle/_ref, all host cores) on a bounded 32-token sample of the step.
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_04984_b200 import meft as G  # noqa: E402

D = 4096


def run_point(ctx, T, M, N, K, kk=4, steps=5, warmup=2):
    st = G.Store(ctx, 1, D, M, N, G.STORE_MIXED)
    b = 1.0 / D ** 0.5
    gen = torch.Generator(device="cuda").manual_seed(1)
    with torch.no_grad():
        for name in ("w_a", "w_b", "w_g"):
            w = st.tensor(0, name)
            w.uniform_(-b, b, generator=gen)
            c = st.tensor(0, name + "_compute")
            for r0 in range(0, w.shape[0], 65536):  # chunked: no full-size bf16 temporary
                c[r0:r0 + 65536].copy_(w[r0:r0 + 65536].to(torch.bfloat16))
    h = (torch.rand((T, D), generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16)
    g = (torch.rand((T, D), generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16)
    ctx.set_timing(True)
    info = None
    for _ in range(warmup):
        info = st.layer_step(0, h, g, kk, K, 1e-4)
    torch.cuda.synchronize()
    ctx.read_timing()  # drop the warm-up phases
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sizes = []
    for _ in range(steps):
        info = st.layer_step(0, h, g, kk, K, 1e-4)
        sizes.append(info["union_size"])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    phases = ctx.read_timing()
    ctx.set_timing(False)
    S = sum(sizes) / len(sizes)
    flops = 12.0 * T * D * S
    line = {"T": T, "M": M, "experts": N, "K": K, "kk": kk, "union": S, "ms_per_step": ms, "tokens_per_s": T / ms * 1e3,
            "ffn_tflops": flops / (ms * 1e-3) / 1e12,
            "phases_ms": {k: v[0] / steps for k, v in phases.items()},
            "store_gb": (6 * 4 + 2 * 2) * M * D / 1e9}
    st.close()
    del h, g
    torch.cuda.empty_cache()
    return line


def cpu_point(T, M, N, K, kk=4, tokens=32):
    """The reference's ref_layer_step (meft_ffn -> sparse_backward -> scatter_grads -> sparse_adam_update) on the
    point's geometry for a bounded token sample; returns tokens/s and the thread count."""
    import numpy as np

    from oracle import oracle as O

    R = O.ref()
    cores = os.cpu_count()
    R.ref_set_threads(cores)
    st = O.RefStore(1, D, M, N, seed=1)
    rng = np.random.default_rng(7)
    st.set(0, "w_b", rng.uniform(-1, 1, size=(M, D)) / D ** 0.5)
    h = rng.uniform(-1, 1, size=(tokens, D))
    g = rng.uniform(-1, 1, size=(tokens, D))
    st.layer_step(0, h[:2], g[:2], kk, K, 1e-4, want_outputs=False)  # warm-up
    t0 = time.perf_counter()
    st.layer_step(0, h, g, kk, K, 1e-4, want_outputs=False)
    return tokens / (time.perf_counter() - t0), cores


def main():
    args = sys.argv[1:]
    T = 8192
    if args and ":" not in args[0]:
        T = int(args[0])
        args = args[1:]
    ctx = G.Context(0)
    for spec in args or ["65536:256:128"]:
        M, N, K = (int(x) for x in spec.split(":"))
        try:
            line = run_point(ctx, T, M, N, K)
            if os.environ.get("MEFT_SWEEP_CPU") == "1" and M <= 65536:
                tps, cores = cpu_point(T, M, N, K)
                line["cpu_reference"] = {"tokens_per_s": tps, "cores": cores, "sample_tokens": 32,
                                         "gpu_over_cpu": line["tokens_per_s"] / tps}
            print(json.dumps(line), flush=True)
        except Exception as e:  # e.g. a point that does not fit HBM
            print(json.dumps({"T": T, "M": M, "experts": N, "K": K, "error": str(e)[:300]}), flush=True)
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
