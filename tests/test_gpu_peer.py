"""Fused reduce-scatter over peer memory (EPI_PEER_F32 + meft_peer_reduce), data path checked at P = 4 inside ONE
process: four emulated ranks, each with its own expert shard, push their out / grad_h rows into four local
buffers that stand in for the homes' peer-mapped receive buffers (no rank ever waits on another). Folding each
home's slots must equal the per-rank partial sums added in slot order -- bit for bit."""
import ctypes as C

import numpy as np
import pytest
import torch

from paper_2406_04984_b200 import _lib
from paper_2406_04984_b200 import meft as G
from paper_2406_04984_b200 import sharded as SH

pytestmark = pytest.mark.gpu


def _shard_store(ctx, d, m_loc, n_loc, seed):
    st = G.Store(ctx, 1, d, m_loc, n_loc, G.STORE_MIXED)
    gen = torch.Generator(device="cuda").manual_seed(seed)
    b = 1.0 / d ** 0.5
    for name in ("w_a", "w_b", "w_g"):
        w = st.tensor(0, name)
        w.uniform_(-b, b, generator=gen)
        st.tensor(0, name + "_compute").copy_(w.to(torch.bfloat16))
    return st


def test_peer_push_and_fold_equals_reduce_scatter(ctx):
    P, T, d, m_loc, n_loc = 4, 128, 512, 1024, 16
    gen = torch.Generator(device="cuda").manual_seed(3)
    h_all = (torch.rand((P * T, d), generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16)
    g_all = (torch.rand((P * T, d), generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16)
    unions = [torch.sort(torch.randperm(m_loc, generator=torch.Generator().manual_seed(10 + r))[:700]).values
              .to(torch.int32).cuda() for r in range(P)]
    # reference: local partial sums of every rank, reduce-scattered by hand (slot order)
    parts = []
    for r in range(P):
        st = _shard_store(ctx, d, m_loc, n_loc, 100 + r)
        eng = SH.DeviceEngine(ctx, st, st.tensor(0, "w_g_compute"))
        parts.append(eng.ffn_local(h_all, g_all, unions[r], 1e-3))
    torch.cuda.synchronize()
    # peer path: the same shards (fresh stores), rows pushed into the homes' buffers
    bufs = [(torch.zeros((P, T, d), dtype=torch.float32, device="cuda"),
             torch.zeros((P, T, d), dtype=torch.float32, device="cuda")) for _ in range(P)]
    bases = [(o.data_ptr(), gh.data_ptr()) for o, gh in bufs]
    xs = [SH.PeerExchange(ctx, T, d, world=P, rank=r, local=bases) for r in range(P)]
    for r in range(P):
        st = _shard_store(ctx, d, m_loc, n_loc, 100 + r)
        eng = SH.DeviceEngine(ctx, st, st.tensor(0, "w_g_compute"))
        assert eng.ffn_local(h_all, g_all, unions[r], 1e-3, peer=xs[r]) == (None, None)
    torch.cuda.synchronize()
    for home in range(P):
        rows = slice(home * T, (home + 1) * T)
        for which in (0, 1):
            want = parts[0][which][rows].clone()
            for r in range(1, P):
                want += parts[r][which][rows]
            got = xs[home].reduce(ctx, which)
            torch.cuda.synchronize()
            assert torch.equal(got, want), (home, which)
    # slot s of home h holds exactly rank s's rows of that home
    assert torch.equal(bufs[2][0][1], parts[1][0][2 * T:3 * T])


def test_peer_push_with_an_empty_local_union_zeroes_its_slots(ctx):
    """A rank that owns none of the selected pairs (empty local union) must still overwrite its slot in every home's
    receive buffer with zeros -- the buffers are reused across steps, so a skipped slot would fold stale rows of the
    previous step into out / grad_h -- and must still fire grad_h_done (the overlapped copy / fold waits on it)."""
    P, T, d, m_loc, n_loc = 2, 64, 256, 512, 8
    gen = torch.Generator(device="cuda").manual_seed(5)
    h_all = (torch.rand((P * T, d), generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16)
    g_all = (torch.rand((P * T, d), generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16)
    unions = [torch.arange(0, m_loc, 3, dtype=torch.int32, device="cuda"),
              torch.empty(0, dtype=torch.int32, device="cuda")]  # rank 1 owns nothing this step
    st0 = _shard_store(ctx, d, m_loc, n_loc, 300)
    want = SH.DeviceEngine(ctx, st0, st0.tensor(0, "w_g_compute")).ffn_local(h_all, g_all, unions[0], 1e-3)
    # receive buffers full of garbage from a "previous step"
    bufs = [(torch.full((P, T, d), 7.0, device="cuda"), torch.full((P, T, d), -3.0, device="cuda")) for _ in range(P)]
    bases = [(o.data_ptr(), gh.data_ptr()) for o, gh in bufs]
    xs = [SH.PeerExchange(ctx, T, d, world=P, rank=r, local=bases) for r in range(P)]
    for r in range(P):
        st = _shard_store(ctx, d, m_loc, n_loc, 300 + r)
        eng = SH.DeviceEngine(ctx, st, st.tensor(0, "w_g_compute"))
        gh_done = torch.cuda.Event()
        gh_done.record()
        assert eng.ffn_local(h_all, g_all, unions[r], 1e-3, gh_done=gh_done, peer=xs[r]) == (None, None)
        torch.cuda.synchronize()
        assert gh_done.query()
    for home in range(P):
        rows = slice(home * T, (home + 1) * T)
        for which in (0, 1):
            assert torch.equal(bufs[home][which][1], torch.zeros((T, d), device="cuda")), (home, which)
            got = xs[home].reduce(ctx, which)
            torch.cuda.synchronize()
            assert torch.equal(got, want[which][rows] + 0.0), (home, which)


def test_peer_reduce_rejects_bad_arguments(ctx):
    out = torch.empty((4, 8), dtype=torch.float32, device="cuda")
    st = _lib.lib().meft_peer_reduce(ctx.h, C.c_void_p(out.data_ptr()), 9, 1, 32, C.c_void_p(out.data_ptr()))
    assert st == 2


def test_ipc_handle_maps_buffer_in_another_process(ctx, tmp_path):
    """meft_ipc_handle / meft_ipc_open across processes (how PeerExchange maps the homes' receive buffers): a
    child process opens the parent's buffer, writes a pattern through it and exits; the parent reads it back."""
    import os
    import subprocess
    import sys

    n = 1 << 16
    p = C.c_void_p()
    _lib.check(_lib.lib().meft_device_alloc(ctx.h, n * 4, C.byref(p)), ctx.h)
    try:
        hb = (C.c_char * 64)()
        _lib.check(_lib.lib().meft_ipc_handle(ctx.h, p, hb), ctx.h)
        (tmp_path / "h.bin").write_bytes(bytes(hb))
        child = f"""
import ctypes as C, sys, torch
sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})
from paper_2406_04984_b200 import _lib, meft as G
ctx = G.Context(0)
hb = (C.c_char * 64).from_buffer_copy(open({str(tmp_path / "h.bin")!r}, "rb").read())
q = C.c_void_p()
_lib.check(_lib.lib().meft_ipc_open(ctx.h, hb, C.byref(q)), ctx.h)
t = torch.as_tensor(G._CAI(q.value, ({n},), "<f4"), device="cuda:0")
t.copy_(torch.arange({n}, dtype=torch.float32, device="cuda:0") * 0.5)
torch.cuda.synchronize()
_lib.check(_lib.lib().meft_ipc_close(ctx.h, q), ctx.h)
"""
        r = subprocess.run([sys.executable, "-c", child], capture_output=True, text=True, timeout=240)
        assert r.returncode == 0, r.stderr[-2000:]
        got = torch.as_tensor(G._CAI(p.value, (n,), "<f4"), device="cuda:0")
        assert torch.equal(got, torch.arange(n, dtype=torch.float32, device="cuda:0") * 0.5)
    finally:
        _lib.lib().meft_device_free(ctx.h, p)
