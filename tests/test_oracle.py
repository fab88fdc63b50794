"""Pins the CPU oracle (oracle/meft_oracle.c) before anything is checked against it.

(1) against golden fixtures produced by the UNMODIFIED reference (oracle/gen_golden.py), and
(2) against the known-answer tests of proj/tests/test_{adapter,experts,memtier}.cpp, restated here.
When the reference build (oracle/_ref) is present, it is also compared live on fresh seeds.
"""
import numpy as np
import pytest

from oracle import oracle as O


def test_rng_matches_reference_fixture(golden):
    g = golden("rng.npz")
    for (s, t), m, draws in zip(g["seeds"], g["mixed"], g["draws"]):
        assert O.mix_seed(int(s), int(t)) == int(m)
        np.testing.assert_array_equal(O.uniform(int(m), (64,), -0.5, 0.25), draws)


def _sel_inputs(T, d, r, N, seed, bf16):
    mk = lambda s, shape: O.uniform(O.mix_seed(seed, s), shape, -1.0, 1.0)  # noqa: E731
    h, w_a, w_g = mk(1, (T, d)), mk(2, (d, r)), mk(3, (N, d))
    if bf16:
        h, w_a, w_g = O.bf16_round(h), O.bf16_round(w_a), O.bf16_round(w_g)
    return h, w_a, w_g


@pytest.mark.parametrize("name", ["cfg1_bf16", "cfg1_f64", "odd_d_f64", "clamp", "full_budget", "one_expert"])
def test_ke_select_matches_reference_fixture(golden, name):
    g = golden("selection.npz")
    f = lambda k: g[f"{name}__{k}"]  # noqa: E731
    T, d, r, N, kk, k = (int(f(x)) for x in ("T", "d", "r", "N", "kk", "k"))
    h, w_a, w_g = _sel_inputs(T, d, r, N, int(f("seed")), bool(f("bf16")))
    res = O.ke_select(h, w_g, w_a, kk, k)
    np.testing.assert_array_equal(res["per_token"], f("per_token"))
    np.testing.assert_array_equal(res["tau"], f("tau"))
    np.testing.assert_array_equal(res["unioned"], f("unioned"))
    assert res["take"] == int(f("take"))
    flat = O.topk_select(h, w_a, k)
    np.testing.assert_array_equal(flat["per_token"], f("flat_per_token"))
    np.testing.assert_array_equal(flat["unioned"], f("flat_unioned"))


def test_ffn_matches_reference_fixture(golden):
    g = golden("ffn.npz")
    for i in range(int(g["n"])):
        c = lambda k: g[f"c{i}__{k}"]  # noqa: E731
        n = c("w_in").shape[1]
        w_in, w_out = (c("w_in"), c("w_out")) if n else (None, None)
        wak, wbk = O.gather_adapter(c("w_a"), c("w_b"), c("S"))
        out, z, pre = O.ffn_forward(c("h"), wak, wbk, w_in, w_out, int(c("act")))
        np.testing.assert_array_equal(z, c("z"))
        np.testing.assert_allclose(out, c("out"), rtol=1e-13, atol=1e-14)
        gwa, gwb, gh = O.ffn_backward(c("G"), c("h"), z, pre if n else None, wak, wbk, w_in, w_out, int(c("act")))
        np.testing.assert_allclose(gwa, c("gwa"), rtol=1e-13, atol=1e-14)
        np.testing.assert_allclose(gwb, c("gwb"), rtol=1e-13, atol=1e-14)
        np.testing.assert_allclose(gh, c("gh"), rtol=1e-12, atol=1e-13)


def test_scatter_adam_matches_reference_fixture(golden):
    g = golden("adam.npz")
    st = O.OracleStore(g["w_a0"], g["w_b0"])
    for i in range(int(g["steps"])):
        s = lambda k: g[f"s{i}__{k}"]  # noqa: E731
        st.scatter_grads(s("S"), s("ga"), s("gb"))
        st.sparse_adam(float(s("lr")))
        for name in ("w_a", "w_b", "m_a", "v_a", "m_b", "v_b"):
            np.testing.assert_allclose(getattr(st, name), s(name), rtol=1e-14, atol=1e-17, err_msg=name)
        np.testing.assert_array_equal(st.pair_step, s("pair_step"))


# ---------------------------------------------------------------- reference known-answer tests (restated)

def test_topk_zero_input_ties_to_low_indices():  # test_adapter.cpp:93-99
    res = O.topk_select(np.zeros((2, 3)), np.zeros((3, 6)), 3)
    assert res["per_token"].tolist() == [[0, 1, 2], [0, 1, 2]]
    assert res["unioned"].tolist() == [0, 1, 2]


def test_topk_scores_example():  # test_adapter.cpp:101-117
    w_a = np.array([[1.0, 0.0, -1.0, 0.5], [0.0, 1.0, 0.0, 0.5]])
    res = O.topk_select(np.array([[1.0, 2.0]]), w_a, 2)
    assert res["unioned"].tolist() == [1, 3]


def test_topk_clamp_and_invalid():  # test_adapter.cpp:119-128
    w_a = O.uniform(5, (2, 3), -1, 1)
    res = O.topk_select(O.uniform(6, (1, 2), -1, 1), w_a, 10)
    assert res["warned"] and len(res["unioned"]) == 3
    with pytest.raises(O.OracleError):
        O.topk_select(O.uniform(6, (1, 2), -1, 1), w_a, 0)


def test_union_bound():  # test_adapter.cpp:139-152
    for it in range(20):
        rs = np.random.RandomState(it)
        d, r, T, k = rs.randint(1, 5), rs.randint(1, 13), rs.randint(1, 13), rs.randint(1, 13)
        res = O.topk_select(O.uniform(it, (T, d), -1, 1), O.uniform(it + 100, (d, r), -1, 1), k)
        assert len(res["unioned"]) <= min(r, T * k)


def test_gather_validation():  # test_adapter.cpp:154-176
    w_a, w_b = O.uniform(8, (3, 4), -1, 1), O.uniform(9, (4, 3), -1, 1)
    wak, wbk = O.gather_adapter(w_a, w_b, [0, 1, 2, 3])
    np.testing.assert_array_equal(wak, w_a)
    np.testing.assert_array_equal(wbk, w_b)
    with pytest.raises(O.OracleError) as e:
        O.gather_adapter(w_a, w_b, [2, 0])
    assert e.value.code == 2
    with pytest.raises(O.OracleError) as e:
        O.gather_adapter(w_a, w_b, [7])
    assert e.value.code == 3 and "7" in str(e.value)


def test_route_and_select_experts():  # test_experts.cpp:24-49
    w_g = np.array([[1.0, 0.0], [0.0, 1.0]])
    np.testing.assert_allclose(O.route_scores(np.array([0.3, 0.7]), w_g), [0.3, 0.7])
    assert O.select_experts([0.3, 0.7], 1).tolist() == [1]
    assert O.select_experts([1.0, 1.0, 1.0, 1.0], 2).tolist() == [0, 1]
    assert O.select_experts([0.5, -0.5, 0.25], 3).tolist() == [0, 1, 2]
    assert O.select_experts([0.5, -0.5], 10).tolist() == [0, 1]
    with pytest.raises(O.OracleError):
        O.select_experts([0.5], 0)


def test_ke_select_degenerate_equivalences():  # test_experts.cpp:59-85
    w_a = O.uniform(21, (4, 12), -1, 1)
    h = O.uniform(22, (6, 4), -1, 1)
    a = O.ke_select(h, O.uniform(23, (1, 4), -1, 1), w_a, 1, 4)
    b = O.topk_select(h, w_a, 4)
    np.testing.assert_array_equal(a["per_token"], b["per_token"])
    c = O.ke_select(h, O.uniform(24, (4, 4), -1, 1), w_a, 4, 3)
    d = O.topk_select(h, w_a, 3)
    np.testing.assert_array_equal(c["per_token"], d["per_token"])


def test_ke_select_routing_restricts():  # test_experts.cpp:87-110
    w_a = np.zeros((2, 4))
    w_a[0, 0], w_a[0, 2], w_a[0, 3] = 100.0, 1.0, 2.0
    w_g = np.zeros((2, 2))
    w_g[0, 0], w_g[1, 0] = -1.0, 1.0
    res = O.ke_select(np.array([[1.0, 0.0]]), w_g, w_a, 1, 1)
    assert res["unioned"].tolist() == [3]


def test_adam_first_step_closed_form():  # test_memtier.cpp:136-156
    st = O.OracleStore(O.uniform(99, (3, 6), -0.5, 0.5), np.zeros((6, 3)))
    w0, g, lr = st.w_a[1, 2], 0.42, 3e-3
    ga = np.zeros((3, 1))
    ga[1, 0] = g
    st.scatter_grads([2], ga, np.zeros((1, 3)))
    st.sparse_adam(lr)
    assert st.w_a[1, 2] == pytest.approx(w0 - lr * g / (abs(g) + 1e-8), rel=1e-12)
    assert st.pair_step.tolist() == [0, 0, 1, 0, 0, 0]


@pytest.mark.skipif(not O.ref_available(), reason="reference build (oracle/_ref) not present")
@pytest.mark.parametrize("seed", [101, 102, 103])
def test_oracle_vs_live_reference(seed):
    rs = np.random.RandomState(seed)
    T, d, N = rs.randint(1, 40), rs.randint(1, 40), rs.randint(1, 9)
    r = N * rs.randint(1, 12)
    kk, k = rs.randint(1, N + 2), rs.randint(1, 20)
    h, w_a, w_g = _sel_inputs(T, d, r, N, seed, bool(seed % 2))
    a, b = O.ke_select(h, w_g, w_a, kk, k), O.ref_ke_select(h, w_g, w_a, kk, k)
    for key in ("per_token", "tau", "unioned"):
        np.testing.assert_array_equal(a[key], b[key])
    wak, wbk = O.gather_adapter(w_a, O.uniform(seed, (r, d), -1, 1), a["unioned"])
    o1, z1, _ = O.ffn_forward(h, wak, wbk)
    o2, z2, _ = O.ref_ffn_forward(h, wak, wbk)
    np.testing.assert_array_equal(z1, z2)
    np.testing.assert_allclose(o1, o2, rtol=1e-13, atol=1e-14)
