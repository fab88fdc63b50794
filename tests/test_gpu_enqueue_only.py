"""The enqueue-only layer step (meft_ctx_set_host_sync(ctx, 0), include/meft_cuda.h) and CUDA-graph capture of it.

With host sync off the fused step never reads |S| back: the six FFN GEMMs are launched for the capacity M and read
the union size from device memory before their first tile (GemmEpilogue::extent / apply_extent in gemm_sm100.cu),
the Adam coefficient and key-statistics kernels likewise. The claim is BIT-identity with the synchronising step,
which sizes every launch on the host: selection, out, grad_h and all tables / moments / counters, over several
steps (so the refreshed key statistics feed the next selection), on shapes that exercise both GEMM kernels (1-CTA
and CTA pair), unions that are not multiples of 64 or 256, and MIXED / COMPACT stores. A capture into a CUDA graph
succeeds only if the step neither synchronises nor allocates (thread-local capture mode makes either an error), and
the replayed graph must match the eager synchronising step bit for bit on fresh inputs."""
import numpy as np
import pytest
import torch

from paper_2406_04984_b200 import meft as G

pytestmark = pytest.mark.gpu

TABLES = ("w_a", "w_b", "m_a", "v_a", "m_b", "v_b", "pair_step", "w_a_compute", "w_b_compute")


def _store(ctx, d, M, N, seed, prec=G.STORE_MIXED, layers=1):
    st = G.Store(ctx, layers, d, M, N, prec)
    b = 1.0 / d ** 0.5
    for layer in range(layers):
        st.upload(layer, "w_a", G.reference_uniform(seed + layer, 0x5000, (d, M), -b, b, bf16=True))
        st.upload(layer, "w_g", G.reference_uniform(seed + layer, 0x5001, (N, d), -b, b, bf16=True))
        st.upload(layer, "w_b", G.reference_uniform(seed + layer, 0x7001, (M, d), -b, b, bf16=True))
    return st


def _inputs(T, d, step):
    h = torch.from_numpy(G.reference_uniform(11, 0x7002 + step, (T, d), -1, 1, bf16=True)).cuda().bfloat16()
    g = torch.from_numpy(G.reference_uniform(11, 0x7003 + step, (T, d), -1, 1, bf16=True)).cuda().bfloat16()
    return h, g


def _assert_tables_equal(a, b, layers=1):
    for layer in range(layers):
        for name in TABLES:
            ta, tb = a.tensor(layer, name), b.tensor(layer, name)
            assert torch.equal(ta.view(torch.int8) if ta.dtype == torch.bfloat16 else ta,
                               tb.view(torch.int8) if tb.dtype == torch.bfloat16 else tb), (layer, name)


@pytest.fixture(scope="module")
def ctxs():
    sync, free = G.Context(0), G.Context(0)
    sync.set_host_sync(True)
    free.set_host_sync(False)
    yield sync, free
    free.close()
    sync.close()


@pytest.fixture(scope="module")
def side():
    """Contexts on a non-default stream (the legacy default stream cannot be captured): (host sync on, off)."""
    s = torch.cuda.Stream()
    sync, free = G.Context(0, stream=s), G.Context(0, stream=s)
    sync.set_host_sync(True)
    free.set_host_sync(False)
    yield sync, free
    free.close()
    sync.close()


# (d, M, N, K, T, precision, gather): cfg1 (the reference's own workload: 1-CTA GEMMs), a pair-kernel shape whose
# union is well below M and not a multiple of 64, an odd token count, a COMPACT store -- all with the gather the
# step picks ("auto": the kernel here); the same sparse unions with TMA gathers forced (broken runs ->
# tile::gather4, rows past the union -> out-of-bounds zeros); a dense shape where AUTO takes TMA (full union)
SHAPES = [
    (512, 4096, 64, 32, 256, G.STORE_MIXED, "auto"),
    (1024, 16384, 64, 32, 300, G.STORE_MIXED, "auto"),
    (512, 8192, 32, 16, 333, G.STORE_MIXED, "auto"),
    (1024, 16384, 64, 32, 300, G.STORE_COMPACT, "auto"),
    (1024, 16384, 64, 32, 300, G.STORE_MIXED, "tma"),
    (512, 8192, 32, 16, 333, G.STORE_MIXED, "tma"),
    (512, 16384, 64, 128, 2048, G.STORE_MIXED, "auto"),
    (512, 16384, 64, 128, 2048, G.STORE_MIXED, "kernel"),
    (1056, 3300, 33, 40, 200, G.STORE_MIXED, "auto"),   # M not a multiple of 64, d % 256 != 0, 33 experts
    (1056, 3300, 33, 40, 200, G.STORE_MIXED, "tma"),
    (1056, 8192, 32, 64, 384, G.STORE_MIXED, "tma"),   # partial 256-column Adam tiles on the pair kernel
]


@pytest.mark.parametrize("shape", SHAPES, ids=["cfg1", "pair", "odd", "compact", "pair-tma", "odd-tma", "dense",
                                                "dense-kernel", "m3300", "m3300-tma", "d1056-tma"])
def test_enqueue_only_step_is_bit_identical_to_the_synchronising_step(ctxs, shape):
    d, M, N, K, T, prec, gather = shape
    kk, lr = 4, 1e-3
    sync, free = ctxs
    for c in ctxs:
        c.set_gather(gather)
    a, b = _store(sync, d, M, N, 5, prec), _store(free, d, M, N, 5, prec)
    sizes = []
    for step in range(3):
        h, g = _inputs(T, d, step)
        res = []
        for st in (a, b):
            out = torch.full((T, d), float("nan"), device="cuda")
            gh = torch.full((T, d), float("nan"), device="cuda")
            r = st.layer_step(0, h, g, kk, K, lr, out=out, grad_h=gh, want_selection=True)
            res.append((r, out, gh))
        torch.cuda.synchronize()
        (ra, oa, ga), (rb, ob, gb) = res
        assert ra["union_size"] == rb["union_size"] and ra["rescored"] == rb["rescored"]
        assert torch.equal(ra["per_token"], rb["per_token"]) and torch.equal(ra["unioned"], rb["unioned"])
        assert torch.equal(oa, ob) and torch.equal(ga, gb), step
        assert not torch.isnan(ob).any() and not torch.isnan(gb).any()
        _assert_tables_equal(a, b)
        sizes.append(ra["union_size"])
    print(f"\nenqueue-only == synchronising step, shape {shape[:5]} gather {gather}: |S| per step {sizes} (M = {M})")
    assert any(s % 64 for s in sizes) or M == sizes[0]  # the partial-tile paths ran (or the union is full)
    for c in ctxs:
        c.set_gather("auto")
    a.close()
    b.close()


def test_enqueue_only_step_without_info_never_waits(ctxs):
    """want_info=False: no meft_step_info, so nothing is read back; two layers enqueue back to back and match."""
    d, M, N, K, T = 1024, 16384, 64, 32, 300
    sync, free = ctxs
    a, b = _store(sync, d, M, N, 9, layers=2), _store(free, d, M, N, 9, layers=2)
    for step in range(2):
        h, g = _inputs(T, d, 10 + step)
        outs = []
        for st, info in ((a, True), (b, False)):
            o = [torch.empty((T, d), device="cuda") for _ in range(2)]
            for layer in range(2):
                st.layer_step(layer, h, g, 4, K, 1e-3, out=o[layer], want_info=info)
            outs.append(o)
        torch.cuda.synchronize()
        for layer in range(2):
            assert torch.equal(outs[0][layer], outs[1][layer])
    _assert_tables_equal(a, b, layers=2)
    a.close()
    b.close()


@pytest.mark.parametrize("shape", [(512, 4096, 64, 32, 256), (1024, 16384, 64, 32, 300), (512, 16384, 64, 128, 2048)],
                         ids=["cfg1", "pair", "dense-tma"])
def test_graph_of_a_two_layer_step_replays_bit_identically(ctxs, side, shape):
    d, M, N, K, T = shape
    kk, lr, L = 4, 1e-3, 2
    sync, _ = ctxs
    _, free = side  # captured stream; everything else runs on the default stream, synchronised in between
    ref, st = _store(sync, d, M, N, 21, layers=L), _store(free, d, M, N, 21, layers=L)
    torch.cuda.synchronize()
    h_buf = torch.empty((T, d), dtype=torch.bfloat16, device="cuda")
    g_buf = torch.empty_like(h_buf)
    out = [torch.empty((T, d), device="cuda") for _ in range(L)]
    gh = [torch.empty((T, d), device="cuda") for _ in range(L)]
    per = [torch.empty((T, K), dtype=torch.int32, device="cuda") for _ in range(L)]

    def step_free():
        for layer in range(L):
            st.layer_step(layer, h_buf, g_buf, kk, K, lr, out=out[layer], grad_h=gh[layer], per_token=per[layer],
                          want_info=False)

    def step_ref(h, g):
        o = []
        for layer in range(L):
            oo, gg = torch.empty((T, d), device="cuda"), torch.empty((T, d), device="cuda")
            r = ref.layer_step(layer, h, g, kk, K, lr, out=oo, grad_h=gg, want_selection=True)
            o.append((r["per_token"], oo, gg))
        return o

    # step 0 eagerly on both (allocates every scratch buffer), then capture one step and replay it three times
    h, g = _inputs(T, d, 30)
    h_buf.copy_(h)
    g_buf.copy_(g)
    torch.cuda.synchronize()
    step_free()
    step_ref(h, g)
    torch.cuda.synchronize()
    with free.graph() as graph:
        step_free()
    torch.cuda.synchronize()
    for it in range(3):
        h, g = _inputs(T, d, 31 + it)
        h_buf.copy_(h)
        g_buf.copy_(g)
        torch.cuda.synchronize()
        graph.replay()
        r = step_ref(h, g)
        torch.cuda.synchronize()
        for layer in range(L):
            assert torch.equal(per[layer], r[layer][0]), (it, layer)
            assert torch.equal(out[layer], r[layer][1]) and torch.equal(gh[layer], r[layer][2]), (it, layer)
    _assert_tables_equal(ref, st, layers=L)
    graph.close()
    ref.close()
    st.close()


def test_a_synchronising_step_cannot_be_captured(side):
    """Host sync on: the step must refuse to be captured rather than break the capture."""
    sync, _ = side
    d, M, N, K, T = 512, 4096, 64, 32, 256
    st = _store(sync, d, M, N, 3)
    h, g = _inputs(T, d, 40)
    torch.cuda.synchronize()
    st.layer_step(0, h, g, 4, K, 1e-3)  # warm-up
    torch.cuda.synchronize()
    with pytest.raises(G.MeftError, match="cannot be captured"):
        with sync.graph():
            st.layer_step(0, h, g, 4, K, 1e-3)
    # the context still works afterwards
    r = st.layer_step(0, h, g, 4, K, 1e-3)
    torch.cuda.synchronize()
    assert r["union_size"] > 0
    st.close()


def test_capturing_a_step_that_asks_for_its_info_is_refused(side):
    """meft_step_info is read back at the end of an enqueue-only step: while capturing, the step asks for NULL."""
    _, free = side
    d, M, N, K, T = 512, 4096, 64, 32, 256
    st = _store(free, d, M, N, 4)
    h, g = _inputs(T, d, 70)
    torch.cuda.synchronize()
    st.layer_step(0, h, g, 4, K, 1e-3, want_info=False)  # warm-up
    torch.cuda.synchronize()
    with pytest.raises(G.MeftError, match="NULL meft_step_info"):
        with free.graph():
            st.layer_step(0, h, g, 4, K, 1e-3)  # want_info=True
    torch.cuda.synchronize()
    st.close()


def test_enqueue_only_falls_back_outside_the_fused_adam_path(ctxs):
    """Pending scatter_grads take the synchronising path even with host sync off (same results as host sync on)."""
    sync, free = ctxs
    d, M, N, K, T = 512, 4096, 64, 32, 256
    a, b = _store(sync, d, M, N, 13), _store(free, d, M, N, 13)
    S = torch.arange(0, M, 7, dtype=torch.int32, device="cuda")
    gk = torch.full((S.numel(), d), 1e-3, dtype=torch.float32, device="cuda")
    h, g = _inputs(T, d, 50)
    res = []
    for st in (a, b):
        st.scatter_grads(0, S, gk, gk)
        out = torch.empty((T, d), device="cuda")
        r = st.layer_step(0, h, g, 4, K, 1e-3, out=out, want_selection=True)
        res.append((r, out))
    torch.cuda.synchronize()
    assert torch.equal(res[0][1], res[1][1]) and res[0][0]["union_size"] == res[1][0]["union_size"]
    _assert_tables_equal(a, b)
    a.close()
    b.close()
    assert np.isfinite(res[1][1].cpu().numpy()).all()


def test_graph_from_a_cpp_program_linked_only_against_the_c_abi():
    """tests/dropin/graph_capi_check.cpp: the same capture / replay from C++ (no Python), bit for bit."""
    import os
    import subprocess

    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "build", "capi_tests",
                       "graph_capi_check")
    if not os.path.exists(exe):
        pytest.skip("tests/dropin/graph_capi_check.cpp not built (build.build_capi_checks)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "graph_capi_check: OK" in r.stdout


def test_host_buffer_step_with_host_sync_off(ctxs):
    """meft_layer_step_host (pinned host buffers in and out, copies overlapped with the step) on the enqueue-only
    step: the union read-back is deferred to the call's final synchronisation, results equal the default step."""
    d, M, N, K, T = 1024, 16384, 64, 32, 300
    sync, free = ctxs
    a, b = _store(sync, d, M, N, 17), _store(free, d, M, N, 17)
    for step in range(2):
        h, g = _inputs(T, d, 60 + step)
        hh, gg = h.cpu().pin_memory(), g.cpu().pin_memory()
        res = []
        for st in (a, b):
            out = torch.empty((T, d), dtype=torch.float32).pin_memory()
            gh = torch.empty_like(out).pin_memory()
            info = st.layer_step_host(0, hh, gg, 4, K, 1e-3, out_host=out, grad_h_host=gh)
            res.append((info, out, gh))
        assert res[0][0]["union_size"] == res[1][0]["union_size"] > 0
        assert torch.equal(res[0][1], res[1][1]) and torch.equal(res[0][2], res[1][2])
    _assert_tables_equal(a, b)
    a.close()
    b.close()


def test_auto_host_sync_follows_the_read_back_union(ctx):
    """MEFT_HOST_SYNC_AUTO (the default): the first step of a layer reads |S| back; a dense union (one run, >= 3/4
    of M) makes the next steps device-sized -- a capture then succeeds -- while a sparse one keeps the read-back (a
    capture is refused). Results equal the always-synchronising step either way."""
    s = torch.cuda.Stream()
    auto = G.Context(0, stream=s)
    auto.set_host_sync(None)  # MEFT_HOST_SYNC_AUTO (the default unless the environment overrides it)
    sync = G.Context(0, stream=s)
    sync.set_host_sync(True)
    for shape, dense in (((512, 16384, 64, 128, 2048), True), ((512, 4096, 64, 32, 256), False)):
        d, M, N, K, T = shape
        a, b = _store(auto, d, M, N, 23), _store(sync, d, M, N, 23)
        h, g = _inputs(T, d, 80)
        torch.cuda.synchronize()
        for st in (a, b):
            for _ in range(2):
                st.layer_step(0, h, g, 4, K, 1e-3, want_info=False)
        torch.cuda.synchronize()
        if dense:
            with auto.graph() as graph:  # device-sized now: capturable
                a.layer_step(0, h, g, 4, K, 1e-3, want_info=False)
            torch.cuda.synchronize()
            graph.replay()
            b.layer_step(0, h, g, 4, K, 1e-3, want_info=False)
            graph.close()
        else:
            with pytest.raises(G.MeftError, match="cannot be captured"):
                with auto.graph():
                    a.layer_step(0, h, g, 4, K, 1e-3, want_info=False)
        torch.cuda.synchronize()
        _assert_tables_equal(a, b)
        a.close()
        b.close()
    auto.close()
    sync.close()
