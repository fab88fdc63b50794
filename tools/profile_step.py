"""Developer harness: the fused cfg2 layer step alone (for ncu launch lists / captures).
   python tools/profile_step.py [steps] [adam: epilogue|pass] [mixed|compact]
Per step the FFN launches k_gemm_bf16_pair in the order z, out, masked, grad_h, grad W_B, grad W_A."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_04984_b200 import meft as G  # noqa: E402


def make_step(adam="epilogue", prec="mixed"):
    """A cfg2 store and inputs; returns step() running one fused layer step."""
    d, M, N, K, kk, T = 4096, 65536, 256, 128, 4, 8192
    ctx = G.Context(0)
    ctx.set_adam(adam)
    st = G.Store(ctx, 1, d, M, N, G.STORE_COMPACT if prec == "compact" else G.STORE_MIXED)
    st.init_reference(seed=1)  # HostStore::init tables, W_B ~ U(+-1/sqrt d) as in bench.py
    gen = torch.Generator(device="cuda").manual_seed(0x7001)
    w_b = (torch.rand((M, d), generator=gen, device="cuda") * 2 - 1) * d ** -0.5
    st.tensor(0, "w_b").copy_(w_b)
    st.tensor(0, "w_b_compute").copy_(w_b.to(torch.bfloat16))
    del w_b
    h = (torch.rand((T, d), generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16)
    g = (torch.rand((T, d), generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16)
    return lambda: st.layer_step(0, h, g, kk, K, 1e-4)


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    adam = sys.argv[2] if len(sys.argv) > 2 else "epilogue"
    prec = sys.argv[3] if len(sys.argv) > 3 else "mixed"
    step = make_step(adam, prec)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for i in range(steps):
        if i == 1:
            e0.record(torch.cuda.current_stream())
        step()
    e1.record(torch.cuda.current_stream())
    torch.cuda.synchronize()
    if steps > 1:
        print(f"layer step ({adam} Adam, {prec}): {e0.elapsed_time(e1) / (steps - 1):.3f} ms")


if __name__ == "__main__":
    main()
