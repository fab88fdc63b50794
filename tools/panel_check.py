"""Developer check: one fused step with |S| > 65536; prints checksums of outputs and updated tables (run with
MEFT_ACT_PANELS=0 and =1: the panelled layout must be bitwise neutral)."""
import hashlib
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_04984_b200 import meft as G  # noqa: E402

d, N, E, T, kk, K = 256, 512, 256, 2048, 4, 512
M = N * E
ctx = G.Context(0)
st = G.Store(ctx, 1, d, M, N, G.STORE_MIXED)
st.init_reference(seed=3)
gen = torch.Generator(device="cuda").manual_seed(9)
w_b = (torch.rand((M, d), generator=gen, device="cuda") * 2 - 1) * d ** -0.5
st.tensor(0, "w_b").copy_(w_b)
st.tensor(0, "w_b_compute").copy_(w_b.to(torch.bfloat16))
h = (torch.rand((T, d), generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16)
g = (torch.rand((T, d), generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16)
out = torch.empty((T, d), dtype=torch.float32, device="cuda")
gh = torch.empty_like(out)
info = None
for _ in range(2):
    info = st.layer_step(0, h, g, kk, K, 1e-3, out=out, grad_h=gh)
torch.cuda.synchronize()
dig = hashlib.sha256()
for t in (out, gh, st.tensor(0, "w_a"), st.tensor(0, "w_b"), st.tensor(0, "m_a"), st.tensor(0, "v_b")):
    dig.update(t.cpu().numpy().tobytes())
print("union", info["union_size"], "sha", dig.hexdigest()[:16])
