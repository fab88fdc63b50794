"""GPU parity of Key-Experts selection (experts.cpp:47-117, adapter.cpp:42-84): indices must be BIT-EXACT
against the oracle (pinned to the reference) on identical inputs."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2406_04984_b200 import meft as G

pytestmark = pytest.mark.gpu


def dev(x, bf16):
    t = torch.from_numpy(np.ascontiguousarray(x))
    return (t.float().to(torch.bfloat16) if bf16 else t.double()).cuda().contiguous()


def gpu_ke(ctx, h, w_g, w_a, kk, k, bf16):
    sel = G.ke_select(ctx, dev(h, bf16), dev(w_g, bf16), dev(w_a.T, bf16), kk, k)
    return sel.per_token.cpu().numpy(), sel.tau.cpu().numpy(), sel.unioned.cpu().numpy(), sel


def inputs(T, d, r, N, seed, bf16):
    mk = lambda s, shape: O.uniform(O.mix_seed(seed, s), shape, -1.0, 1.0)  # noqa: E731
    h, w_a, w_g = mk(1, (T, d)), mk(2, (d, r)), mk(3, (N, d))
    if bf16:
        h, w_a, w_g = O.bf16_round(h), O.bf16_round(w_a), O.bf16_round(w_g)
    return h, w_a, w_g


@pytest.mark.parametrize("name", ["cfg1_bf16", "cfg1_f64", "odd_d_f64", "clamp", "full_budget", "one_expert"])
def test_ke_select_matches_reference_fixture(ctx, golden, name):
    g = golden("selection.npz")
    f = lambda k: g[f"{name}__{k}"]  # noqa: E731
    T, d, r, N, kk, k = (int(f(x)) for x in ("T", "d", "r", "N", "kk", "k"))
    bf16 = bool(f("bf16"))
    h, w_a, w_g = inputs(T, d, r, N, int(f("seed")), bf16)
    per, tau, uni, sel = gpu_ke(ctx, h, w_g, w_a, kk, k, bf16)
    np.testing.assert_array_equal(per, f("per_token"))
    np.testing.assert_array_equal(tau, f("tau"))
    np.testing.assert_array_equal(uni, f("unioned"))
    assert sel.take == int(f("take"))
    flat = G.topk_select(ctx, dev(h, bf16), dev(w_a.T, bf16), k)
    np.testing.assert_array_equal(flat.per_token.cpu().numpy(), f("flat_per_token"))
    np.testing.assert_array_equal(flat.unioned.cpu().numpy(), f("flat_unioned"))


@pytest.mark.parametrize("seed", range(8))
def test_ke_select_random_shapes_vs_oracle(ctx, seed):
    rs = np.random.RandomState(seed)
    T, d, N = rs.randint(1, 300), rs.randint(1, 70), rs.randint(1, 20)
    r = N * rs.randint(1, 40)
    kk, k = rs.randint(1, N + 3), rs.randint(1, 64)
    bf16 = seed % 2 == 0
    h, w_a, w_g = inputs(T, d, r, N, 500 + seed, bf16)
    want = O.ke_select(h, w_g, w_a, kk, k)
    per, tau, uni, sel = gpu_ke(ctx, h, w_g, w_a, kk, k, bf16)
    np.testing.assert_array_equal(per, want["per_token"])
    np.testing.assert_array_equal(tau, want["tau"])
    np.testing.assert_array_equal(uni, want["unioned"])
    assert sel.warned == want["warned"]


def test_ties_and_signed_zero_follow_reference_order(ctx):
    # zero input: every score is +-0.0 and ties break to the lowest index (test_adapter.cpp:93-99)
    h = np.zeros((2, 3))
    w_a = np.zeros((3, 6))
    w_a[0, 1] = -1.0  # score of key 1 becomes -0.0 for h == 0: still equal to +0.0
    flat = G.topk_select(ctx, dev(h, False), dev(w_a.T, False), 3)
    assert flat.per_token.cpu().tolist() == [[0, 1, 2], [0, 1, 2]]
    # exact duplicate keys: the lower global index wins inside and across experts
    w_a = np.tile(O.uniform(3, (4, 1), -1, 1), (1, 8))
    w_g = np.ones((4, 4))
    res = G.ke_select(ctx, dev(O.uniform(4, (5, 4), -1, 1), False), dev(w_g, False), dev(w_a.T, False), 2, 3)
    assert res.tau.cpu().tolist() == [[0, 1]] * 5
    assert res.per_token.cpu().tolist() == [[0, 1, 2]] * 5


def test_hand_examples(ctx):
    w_a = np.array([[1.0, 0.0, -1.0, 0.5], [0.0, 1.0, 0.0, 0.5]])  # test_adapter.cpp:101-117
    res = G.topk_select(ctx, dev(np.array([[1.0, 2.0]]), False), dev(w_a.T, False), 2)
    assert res.unioned.cpu().tolist() == [1, 3]
    w_a = np.zeros((2, 4))  # test_experts.cpp:87-110
    w_a[0, 0], w_a[0, 2], w_a[0, 3] = 100.0, 1.0, 2.0
    w_g = np.zeros((2, 2))
    w_g[0, 0], w_g[1, 0] = -1.0, 1.0
    res = G.ke_select(ctx, dev(np.array([[1.0, 0.0]]), False), dev(w_g, False), dev(w_a.T, False), 1, 1)
    assert res.unioned.cpu().tolist() == [3]


def test_route_scores_and_select_experts(ctx):
    h = O.bf16_round(O.uniform(7, (33, 64), -1, 1))
    w_g = O.bf16_round(O.uniform(8, (16, 64), -1, 1))
    p = G.route_scores(ctx, dev(h, True), dev(w_g, True)).cpu().numpy()
    for t in range(33):
        np.testing.assert_array_equal(p[t], O.route_scores(h[t], w_g))  # bitwise: same sequential fp64 chain
    tau = G.select_experts(ctx, torch.from_numpy(p).cuda(), 3).cpu().numpy()
    for t in range(33):
        np.testing.assert_array_equal(tau[t], O.select_experts(p[t], 3))


def test_invalid_arguments_raise_reference_kinds(ctx):
    h = dev(np.zeros((2, 4)), False)
    with pytest.raises(G.MeftError) as e:
        G.ke_select(ctx, h, dev(np.zeros((3, 4)), False), dev(np.zeros((8, 4)), False), 1, 2)  # 3 does not divide 8
    assert e.value.kind == "invalid_argument"
    with pytest.raises(G.MeftError) as e:
        G.ke_select(ctx, h, dev(np.zeros((2, 4)), False), dev(np.zeros((8, 4)), False), 1, 0)
    assert e.value.kind == "invalid_argument"
    with pytest.raises(G.MeftError) as e:
        G.ke_select(ctx, h, dev(np.zeros((2, 5)), False), dev(np.zeros((8, 4)), False), 1, 1)
    assert e.value.kind == "ShapeError"


def test_selection_is_deterministic(ctx):
    h, w_a, w_g = inputs(512, 128, 2048, 32, 77, True)
    a = gpu_ke(ctx, h, w_g, w_a, 4, 16, True)
    b = gpu_ke(ctx, h, w_g, w_a, 4, 16, True)
    for x, y in zip(a[:3], b[:3]):
        np.testing.assert_array_equal(x, y)


# ---------------------------------------------------------------- certified tensor-core selection

def _rand_bf16(gen, shape, scale):
    return ((torch.rand(shape, generator=gen, device="cuda") * 2 - 1) * scale).to(torch.bfloat16).contiguous()


def _both_paths(ctx, h, w_g, keys, kk, k):
    a = G.ke_select(ctx, h, w_g, keys, kk, k)
    ctx.set_selection(exact=True)
    try:
        b = G.ke_select(ctx, h, w_g, keys, kk, k)
    finally:
        ctx.set_selection(exact=False)
    return a, b


@pytest.mark.slow
def test_certified_equals_exact_at_baseline_cfg2(ctx):
    """All 8192 tokens of the LLaMA-shape layer: certified tensor-core selection == fp64 SIMT selection."""
    gen = torch.Generator(device="cuda").manual_seed(5)
    d, M, N, K, kk, T = 4096, 65536, 256, 128, 4, 8192
    h = _rand_bf16(gen, (T, d), 1.0)
    keys = _rand_bf16(gen, (M, d), 1 / 64)
    w_g = _rand_bf16(gen, (N, d), 1 / 64)
    a, b = _both_paths(ctx, h, w_g, keys, kk, K)
    assert torch.equal(a.tau, b.tau)
    assert torch.equal(a.per_token, b.per_token)
    assert torch.equal(a.unioned, b.unioned)


@pytest.mark.parametrize("seed", range(4))
def test_certified_resolves_forced_near_ties(ctx, seed):
    """Duplicate and 1-ulp-apart keys/experts force every boundary decision through exact re-scoring;
    a few tokens mix huge and tiny coordinates so the exactness certificate fails and the sequential fp64
    chain is used. The result must still equal the oracle bit for bit."""
    rs = np.random.RandomState(seed)
    T, d, N, E, kk, k = 96, 64, 8, 32, 3, 20
    M = N * E
    w_a = O.bf16_round(rs.uniform(-1, 1, (d, M)) / 8)
    w_a[:, 1::2] = w_a[:, 0::2]                      # exact duplicate keys inside each expert
    w_a[0, 2::4] = O.bf16_round(w_a[0, 2::4] * (1 + 2.0 ** -7))  # neighbours one bf16 ulp apart
    w_g = O.bf16_round(rs.uniform(-1, 1, (N, d)) / 8)
    w_g[1] = w_g[0]                                   # duplicate experts: router ties
    h = O.bf16_round(rs.uniform(-1, 1, (T, d)))
    h[:8, 0] = 1.0
    h[:8, 1:] = O.bf16_round(h[:8, 1:] * 2.0 ** -70)  # products 2^70 apart: certificate fails
    want = O.ke_select(h, w_g, w_a, kk, k)
    for exact in (False, True):
        ctx.set_selection(exact=exact)
        try:
            per, tau, uni, _ = gpu_ke(ctx, h, w_g, w_a, kk, k, True)
        finally:
            ctx.set_selection(exact=False)
        np.testing.assert_array_equal(tau, want["tau"])
        np.testing.assert_array_equal(per, want["per_token"])
        np.testing.assert_array_equal(uni, want["unioned"])


def test_certified_flat_topk(ctx):
    h, w_a, _ = inputs(200, 256, 4096, 1, 91, True)
    want = O.topk_select(h, w_a, 48)
    flat = G.topk_select(ctx, dev(h, True), dev(w_a.T, True), 48)
    np.testing.assert_array_equal(flat.per_token.cpu().numpy(), want["per_token"])
    np.testing.assert_array_equal(flat.unioned.cpu().numpy(), want["unioned"])


@pytest.mark.parametrize("scale_h,scale_k", [(2.0 ** -60, 2.0 ** -75), (2.0 ** 55, 2.0 ** 60), (2.0 ** -130, 1.0),
                                             (1.0, 2.0 ** 62)])
def test_certified_at_extreme_magnitudes(ctx, scale_h, scale_k):
    """Operand scales that push bf16 products to fp32's subnormal range (LSB near 2^-149 and below) or close to
    its overflow: the fp32-product fast paths must step aside exactly when they cannot be exact, and the indices
    must equal the oracle bit for bit. Duplicate keys keep exact re-scoring busy."""
    rs = np.random.RandomState(11)
    T, d, N, E, kk, k = 64, 128, 8, 32, 3, 24
    M = N * E
    w_a = O.bf16_round(rs.uniform(-1, 1, (d, M)) * scale_k)
    w_a[:, 1::2] = w_a[:, 0::2]
    w_g = O.bf16_round(rs.uniform(-1, 1, (N, d)))
    h = O.bf16_round(rs.uniform(-1, 1, (T, d)) * scale_h)
    h[:4, 3:] = O.bf16_round(h[:4, 3:] * 2.0 ** -40)  # wide dynamic range inside a few rows
    want = O.ke_select(h, w_g, w_a, kk, k)
    per, tau, uni, _ = gpu_ke(ctx, h, w_g, w_a, kk, k, True)
    np.testing.assert_array_equal(tau, want["tau"])
    np.testing.assert_array_equal(per, want["per_token"])
    np.testing.assert_array_equal(uni, want["unioned"])


@pytest.mark.parametrize("d", [64, 1024, 4096])
def test_exact_scores_uncertifiable_dots_match_reference_chain(ctx, d):
    """Dots whose products span far more than 53 bits fail the whole-row exactness certificate and take the
    chunked sequential fallback: 128-term chunks whose prefix sums are provably exact are added as one warp sum,
    the rest replay the reference's dependent fp64 chain. Magnitude patterns put the tiny and huge products in the
    same chunk, in different chunks, at chunk edges and at random; every score must equal the reference's dot()
    (kernels.hpp:37-41, via the C restatement) bit for bit."""
    from paper_2406_04984_b200 import sharded as SH
    rs = np.random.RandomState(d)
    M, N, R = 64, 8, 24
    keys = rs.uniform(-1, 1, (M, d))
    rows = rs.uniform(-1, 1, (R, d))
    rows[0, d // 2:] *= 2.0 ** -70                    # tiny tail
    rows[1, :d // 2] *= 2.0 ** -70                    # tiny head
    rows[2, ::2] *= 2.0 ** -60                        # alternating inside every chunk
    rows[3, (np.arange(d) // 128) % 2 == 1] *= 2.0 ** -80  # alternating chunks
    rows[4, 127::128] *= 2.0 ** 40                    # chunk-edge spikes
    rows[5, rs.rand(d) < 0.1] *= 2.0 ** -100           # sparse tiny entries
    rows[6] *= 2.0 ** (rs.randint(-90, 30, d))         # random exponents per entry
    rows[7, : d // 4] = 0.0                           # leading zeros, then a wide range
    rows[7, d // 4:] *= 2.0 ** rs.randint(-70, 0, d - d // 4)
    keys[1::3] *= 2.0 ** (rs.randint(-40, 40, (len(keys[1::3]), d)))
    keys, rows = O.bf16_round(keys), O.bf16_round(rows)
    st = G.Store(ctx, 1, d, M, N, G.STORE_MIXED)
    st.upload(0, "w_a", keys.T.copy())
    st.upload(0, "w_g", O.bf16_round(rs.uniform(-1, 1, (N, d))))
    eng = SH.DeviceEngine(ctx, st, st.tensor(0, "w_g_compute"))
    pr, pk = np.meshgrid(np.arange(R), np.arange(M), indexing="ij")
    got = eng.exact(dev(rows, True), torch.from_numpy(pr.ravel().astype(np.int32)).cuda(),
                    torch.from_numpy(pk.ravel().astype(np.int32)).cuda()).cpu().numpy().reshape(R, M)
    want = np.stack([O.route_scores(rows[r], keys) for r in range(R)])
    np.testing.assert_array_equal(got, want)
