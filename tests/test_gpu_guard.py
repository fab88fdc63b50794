"""Guard zones (MEFT_GUARD_ZONES=1, csrc/meft_capi.cu): this pool does not allow compute-sanitizer, so the library
can put a 4 KB 0xA5 guard after every scratch buffer and every store table and verify them after each C-ABI call.
Here: a guarded run of the hot path (fused MIXED / COMPACT layer steps, the C-ABI sharded step) completes, and a
deliberate one-byte write past a table is caught and named. (The whole -m gpu suite is also run with the variable
set: profiles/r2_guard_zones_suite.txt.)"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import ctypes as C, sys
sys.path.insert(0, {root!r})
import torch
from paper_2406_04984_b200 import meft as G, sharded as SH, _lib
d, M, N, K, kk, T = 512, 4096, 64, 32, 4, 256
ctx = G.Context(0)
def store(prec):
    st = G.Store(ctx, 1, d, M, N, prec)
    b = 1.0 / d ** 0.5
    st.upload(0, "w_a", G.reference_uniform(1, 0x5000, (d, M), -b, b, bf16=True))
    st.upload(0, "w_g", G.reference_uniform(1, 0x5001, (N, d), -b, b, bf16=True))
    st.upload(0, "w_b", G.reference_uniform(1, 0x7001, (M, d), -b, b, bf16=True))
    return st
h = torch.from_numpy(G.reference_uniform(1, 0x7002, (T, d), -1, 1, bf16=True)).cuda().bfloat16()
for prec in (G.STORE_MIXED, G.STORE_COMPACT):
    st = store(prec)
    for _ in range(2):
        st.layer_step(0, h, h, kk, K, 1e-3)
sh = store(G.STORE_MIXED)
layer = SH.CShardedLayer(ctx, sh, sh.tensor(0, "w_g_compute").clone())
layer.step(h, h, kk, K, 1e-3)
torch.cuda.synchronize()
print("guarded run ok", flush=True)
if {poke}:
    w = st.tensor(0, "w_a")  # one byte past the end of the fp32 key table lands in its guard
    end = w.data_ptr() + w.numel() * 4
    rc = _lib.lib().meft_memset(ctx.h, C.c_void_p(end), 0, 1)
    print("poke status", rc, _lib.lib().meft_last_error(ctx.h).decode(), flush=True)
"""


def _run(poke):
    env = dict(os.environ, MEFT_GUARD_ZONES="1")
    return subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, poke=poke)], capture_output=True, text=True,
                          timeout=600, env=env)


def test_guarded_hot_path_has_no_out_of_bounds_writes():
    r = _run(False)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "guarded run ok" in r.stdout


def test_guard_zone_catches_a_write_past_a_table():
    r = _run(True)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [x for x in r.stdout.splitlines() if x.startswith("poke status")][0]
    assert "guard zone after store" in line and "overwritten" in line and not line.startswith("poke status 0")
