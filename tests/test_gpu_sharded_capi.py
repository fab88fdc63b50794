"""The expert-sharded layer step behind the C ABI (meft_layer_step_sharded, csrc/sharded_step.cu): the protocol
issued inside libmeft_cuda.so, over the library's own NCCL communicator or over host callbacks.

  * world 1 over NCCL (the library creates the communicator from its own unique id): bit for bit the single-GPU
    meft_layer_step -- selection, out, grad_h, and every updated table, over two steps
  * P = 2, 4, 8 ranks emulated in one process (one thread + context per rank, the host-callback communicator; no
    kernel waits on another rank): against the single-GPU fused step on the same P*T tokens, the selection and the
    shards' updated tables bit for bit, out / grad_h to fp32 round-off (partials are summed per rank)
  * a C++ program linked only against libmeft_cuda.so runs the world-1 NCCL step and compares it with
    meft_layer_step (tests/dropin/sharded_capi_check.cpp)"""
import os
import subprocess
import threading

import numpy as np
import pytest
import torch

from paper_2406_04984_b200 import meft as G
from paper_2406_04984_b200 import sharded as SH

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _full_store(ctx, d, M, N, seed=1):
    st = G.Store(ctx, 1, d, M, N, G.STORE_MIXED)
    b = 1.0 / d ** 0.5
    st.upload(0, "w_a", G.reference_uniform(seed, 0x5000, (d, M), -b, b, bf16=True))
    st.upload(0, "w_g", G.reference_uniform(seed, 0x5001, (N, d), -b, b, bf16=True))
    st.upload(0, "w_b", G.reference_uniform(seed, 0x7001, (M, d), -b, b, bf16=True))
    return st


def _shard_of(ctx, full, r, P):
    d, M, N = full.d, full.pairs, full.experts
    M_loc, N_loc = M // P, N // P
    sh = G.Store(ctx, 1, d, M_loc, N_loc, G.STORE_MIXED)
    for name in ("w_a", "w_b", "w_a_compute", "w_b_compute"):
        sh.tensor(0, name).copy_(full.tensor(0, name)[r * M_loc:(r + 1) * M_loc])
    return sh


TABLES = ("w_a", "w_b", "m_a", "v_a", "m_b", "v_b", "w_a_compute", "w_b_compute", "pair_step")


def test_capi_sharded_world1_over_nccl_equals_layer_step(ctx):
    d, M, N, K, kk, T, lr = 512, 4096, 64, 32, 4, 256, 1e-3
    ref = _full_store(ctx, d, M, N)
    shard = _full_store(ctx, d, M, N)
    w_g = shard.tensor(0, "w_g_compute").clone()
    layer = SH.CShardedLayer(ctx, shard, w_g)  # world 1: the library's own NCCL communicator
    try:
        for step in range(2):
            h = torch.from_numpy(G.reference_uniform(5, 0x7002 + step, (T, d), -1, 1, bf16=True)).cuda().bfloat16()
            g = torch.from_numpy(G.reference_uniform(5, 0x7003 + step, (T, d), -1, 1, bf16=True)).cuda().bfloat16()
            res = layer.step(h, g, kk, K, lr, want_selection=True)
            out = torch.empty((T, d), dtype=torch.float32, device="cuda")
            gh = torch.empty_like(out)
            want = ref.layer_step(0, h, g, kk, K, lr, out=out, grad_h=gh, want_selection=True)
            torch.cuda.synchronize()
            assert torch.equal(res["per_token"], want["per_token"])
            assert res["union_size"] == want["union_size"]
            assert torch.equal(res["out"], out) and torch.equal(res["grad_h"], gh)
            assert res["peer_path"]  # partial sums stored by the GEMM epilogues into the home's buffers
            assert res["overlap"]  # grad_out all-gathered on a second (split) NCCL communicator and stream
            for n in TABLES:
                assert torch.equal(shard.tensor(0, n), ref.tensor(0, n)), (step, n)
    finally:
        layer.close()


@pytest.mark.parametrize("P", [2, 4, 8])
def test_capi_sharded_multirank_emulated_equals_single_gpu(ctx, P):
    d, M, N, K, kk, T, lr = 512, 4096, 64, 32, 4, 128, 1e-3
    full = _full_store(ctx, d, M, N)
    h = torch.from_numpy(G.reference_uniform(9, 0x7002, (P * T, d), -1, 1, bf16=True)).cuda().bfloat16()
    g = torch.from_numpy(G.reference_uniform(9, 0x7003, (P * T, d), -1, 1, bf16=True)).cuda().bfloat16()
    w_g = full.tensor(0, "w_g_compute").clone()
    shards = [_shard_of(ctx, full, r, P) for r in range(P)]  # before the reference step updates `full`
    out = torch.empty((P * T, d), dtype=torch.float32, device="cuda")
    gh = torch.empty_like(out)
    want = full.layer_step(0, h, g, kk, K, lr, out=out, grad_h=gh, want_selection=True)
    torch.cuda.synchronize()

    tg = SH.ThreadGroup(P)
    results, errors = [None] * P, []

    def rank_main(r):
        try:
            tg.bind(r)
            rctx = G.Context(0)
            layer = SH.CShardedLayer(rctx, shards[r], w_g, group=tg)
            res = layer.step(h[r * T:(r + 1) * T].contiguous(), g[r * T:(r + 1) * T].contiguous(), kk, K, lr,
                             want_selection=True)
            torch.cuda.synchronize()
            results[r] = (res, rctx, layer)
        except Exception as e:  # surfaced below
            errors.append((r, repr(e)))
            tg._barrier.abort()

    threads = [threading.Thread(target=rank_main, args=(r,)) for r in range(P)]
    for t_ in threads:
        t_.start()
    for t_ in threads:
        t_.join(timeout=300)
    assert not errors, errors
    M_loc = M // P
    for r in range(P):
        res = results[r][0]
        rows = slice(r * T, (r + 1) * T)
        assert torch.equal(res["per_token"], want["per_token"][rows])
        assert res["union_size"] == want["union_size"]
        assert res["peer_path"]  # every emulated rank pushed into every home's buffers
        assert float((res["out"] - out[rows]).norm() / out[rows].norm()) < 1e-5
        assert float((res["grad_h"] - gh[rows]).norm() / gh[rows].norm()) < 1e-5
        for n in TABLES:
            assert torch.equal(shards[r].tensor(0, n), full.tensor(0, n)[r * M_loc:(r + 1) * M_loc]), (r, n)
    for r in range(P):
        results[r][2].close()


def test_cpp_program_runs_the_sharded_step_over_nccl(ctx):
    exe = os.path.join(ROOT, "build", "capi_tests", "sharded_capi_check")
    if not os.path.exists(exe):
        pytest.skip("tests/dropin/sharded_capi_check.cpp not built (build.build_capi_checks)")
    for peer in ("1", "0"):  # the reduce-scatter fused into the GEMM epilogues, and the NCCL reduce-scatter fallback
        env = dict(os.environ, MEFT_SHARDED_PEER=peer)
        r = subprocess.run([exe], capture_output=True, text=True, timeout=600, env=env)
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
        assert "sharded_capi_check: OK" in r.stdout
        assert f"peer path {peer}" in r.stdout, r.stdout
        assert "overlap 1" in r.stdout, r.stdout  # grad_out all-gathered on the split communicator's stream


def test_capi_sharded_rank_with_empty_local_union(ctx):
    """Every token routes to rank 0's experts (rank 1 owns nothing that is selected: its local union is empty). Rank
    1 must still return the home rows of out / grad_h (rank 0's contributions only) and leave its tables untouched;
    everything equals the single-GPU step on the same 2*T tokens."""
    P, d, M, N, K, kk, T, lr = 2, 256, 1024, 16, 16, 2, 64, 1e-3
    full = G.Store(ctx, 1, d, M, N, G.STORE_MIXED)
    b = 1.0 / d ** 0.5
    w_g = np.full((N, d), -b)
    w_g[: N // P] = b  # positive hidden states score rank 0's experts above every expert of rank 1
    full.upload(0, "w_g", w_g)
    full.upload(0, "w_a", G.reference_uniform(2, 0x5000, (d, M), -b, b, bf16=True))
    full.upload(0, "w_b", G.reference_uniform(2, 0x7001, (M, d), -b, b, bf16=True))
    h = torch.from_numpy(G.reference_uniform(2, 0x7002, (P * T, d), 0.0, 1.0, bf16=True)).cuda().bfloat16()
    g = torch.from_numpy(G.reference_uniform(2, 0x7003, (P * T, d), -1, 1, bf16=True)).cuda().bfloat16()
    shards = [_shard_of(ctx, full, r, P) for r in range(P)]
    before = {n: shards[1].tensor(0, n).clone() for n in ("w_a", "w_b", "m_a", "pair_step")}
    wg_dev = full.tensor(0, "w_g_compute").clone()
    out = torch.empty((P * T, d), dtype=torch.float32, device="cuda")
    gh = torch.empty_like(out)
    want = full.layer_step(0, h, g, kk, K, lr, out=out, grad_h=gh, want_selection=True)
    torch.cuda.synchronize()
    assert int(want["unioned"].max()) < M // P  # the premise: nothing of rank 1 is selected

    tg = SH.ThreadGroup(P)
    results, errors = [None] * P, []

    def rank_main(r):
        try:
            tg.bind(r)
            rctx = G.Context(0)
            layer = SH.CShardedLayer(rctx, shards[r], wg_dev, group=tg)
            res = layer.step(h[r * T:(r + 1) * T].contiguous(), g[r * T:(r + 1) * T].contiguous(), kk, K, lr,
                             want_selection=True)
            torch.cuda.synchronize()
            results[r] = (res, rctx, layer)
        except Exception as e:  # surfaced below
            errors.append((r, repr(e)))
            tg._barrier.abort()

    threads = [threading.Thread(target=rank_main, args=(r,)) for r in range(P)]
    for t_ in threads:
        t_.start()
    for t_ in threads:
        t_.join(timeout=300)
    assert not errors, errors
    for r in range(P):
        res = results[r][0]
        rows = slice(r * T, (r + 1) * T)
        assert torch.equal(res["per_token"], want["per_token"][rows])
        assert float((res["out"] - out[rows]).norm() / out[rows].norm()) < 1e-5
        assert float((res["grad_h"] - gh[rows]).norm() / gh[rows].norm()) < 1e-5
    for n, t in before.items():
        assert torch.equal(shards[1].tensor(0, n), t), n
    for r in range(P):
        results[r][2].close()
