"""GPU parity of the HBM store: HostStore::init tables, scatter_grads staging and the lazy sparse Adam
(memtier.cpp:60-228) against the reference fixture / oracle."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2406_04984_b200 import meft as G

pytestmark = pytest.mark.gpu


def test_init_reference_tables_bit_identical(ctx):
    st = G.Store(ctx, 2, 48, 96, 8, G.STORE_F64)
    st.init_reference(seed=7)
    b = 1.0 / np.sqrt(48)
    for layer in range(2):
        np.testing.assert_array_equal(st.download(layer, "w_a"), O.uniform(O.mix_seed(7, 0x5000 + 2 * layer), (48, 96), -b, b))
        np.testing.assert_array_equal(st.download(layer, "w_g"), O.uniform(O.mix_seed(7, 0x5001 + 2 * layer), (8, 48), -b, b))
        assert float(np.abs(st.download(layer, "w_b")).max()) == 0.0
        assert st.download(layer, "pair_step").tolist() == [0] * 96
    if O.ref_available():
        ref = O.RefStore(2, 48, 96, 8, seed=7)
        np.testing.assert_array_equal(st.download(1, "w_a"), ref.get(1, "w_a"))


def test_scatter_adam_f64_matches_reference_fixture(ctx, golden):
    g = golden("adam.npz")
    d, r = int(g["d"]), int(g["r"])
    st = G.Store(ctx, 1, d, r, 2, G.STORE_F64)
    st.upload(0, "w_a", g["w_a0"])
    st.upload(0, "w_b", g["w_b0"])
    for i in range(int(g["steps"])):
        s = lambda k: g[f"s{i}__{k}"]  # noqa: E731
        S = torch.tensor(s("S"), dtype=torch.int32, device="cuda")
        st.scatter_grads(0, S, torch.from_numpy(s("ga").T.copy()).cuda(), torch.from_numpy(s("gb")).cuda())
        st.sparse_adam_update(0, float(s("lr")))
        for name in ("w_a", "w_b", "m_a", "v_a", "m_b", "v_b"):
            np.testing.assert_allclose(st.download(0, name), s(name), rtol=1e-14, atol=1e-17, err_msg=name)
        np.testing.assert_array_equal(st.download(0, "pair_step"), s("pair_step"))
        assert float(np.abs(st.download(0, "stage_a")).max()) == 0.0  # staging cleared (memtier.cpp:200-205)
        assert st.download(0, "staged").tolist() == [0] * r


def test_untouched_pairs_bit_identical_and_overlapping_scatters_sum(ctx):  # test_memtier.cpp:76-134
    st = G.Store(ctx, 2, 3, 6, 2, G.STORE_F64)
    st.init_reference(seed=99)
    before = {(l, n): st.download(l, n) for l in range(2) for n in ("w_a", "w_b", "m_a", "v_a")}
    ga = np.zeros((2, 3))
    ga[0, 0] = 0.7
    gb = np.zeros((2, 3))
    gb[1, 2] = -0.3
    st.scatter_grads(1, torch.tensor([0, 3], dtype=torch.int32, device="cuda"), torch.from_numpy(ga).cuda(),
                     torch.from_numpy(gb).cuda())
    st.scatter_grads(1, torch.tensor([3, 3], dtype=torch.int32, device="cuda"), torch.from_numpy(ga).cuda(),
                     torch.from_numpy(ga).cuda())  # repeated index: both entries add, in order
    stage_b = st.download(1, "stage_b")
    np.testing.assert_allclose(stage_b[3], gb[1] + ga[0] + ga[1])  # [3, 3] adds both gradient rows
    st.sparse_adam_update(1, 1e-3)
    ps = st.download(1, "pair_step")
    assert ps.tolist() == [1, 0, 0, 1, 0, 0]
    for (l, n), v in before.items():
        after = st.download(l, n)
        cols = [j for j in range(6) if not (l == 1 and j in (0, 3))]
        if n in ("w_a", "m_a", "v_a"):
            np.testing.assert_array_equal(after[:, cols], v[:, cols])
        else:
            np.testing.assert_array_equal(after[cols, :], v[cols, :])
    with pytest.raises(G.MeftError) as e:
        st.scatter_grads(0, torch.tensor([9], dtype=torch.int32, device="cuda"), torch.zeros((1, 3), dtype=torch.float64,
                         device="cuda"), torch.zeros((1, 3), dtype=torch.float64, device="cuda"))
    assert e.value.kind == "out_of_range"


def test_mixed_store_adam_tolerance(ctx):
    """MIXED store (fp32 master/moments): |dw_gpu - dw_ref| <= 1e-2*lr + 1e-6*|w| over 3 steps."""
    d, r, lr = 64, 32, 1e-3
    w_a = O.bf16_round(O.uniform(1, (d, r), -0.1, 0.1))
    w_b = O.bf16_round(O.uniform(2, (r, d), -0.1, 0.1))
    st = G.Store(ctx, 1, d, r, 4, G.STORE_MIXED)
    st.upload(0, "w_a", w_a)
    st.upload(0, "w_b", w_b)
    orc = O.OracleStore(w_a, w_b)
    for it, S in enumerate([[0, 5, 9], [5, 6, 31], [0, 1, 2, 3, 4, 5]]):
        ga = O.uniform(10 + it, (d, len(S)), -1, 1).astype(np.float32).astype(np.float64)
        gb = O.uniform(20 + it, (len(S), d), -1, 1).astype(np.float32).astype(np.float64)
        st.scatter_grads(0, torch.tensor(S, dtype=torch.int32, device="cuda"),
                         torch.from_numpy(ga.T.copy()).float().cuda(), torch.from_numpy(gb).float().cuda())
        st.sparse_adam_update(0, lr)
        orc.scatter_grads(S, ga, gb)
        orc.sparse_adam(lr)
    for name, want, w0 in (("w_a", orc.w_a, w_a), ("w_b", orc.w_b, w_b)):
        got = st.download(0, name)
        assert np.all(np.abs((got - w0) - (want - w0)) <= 1e-2 * lr + 1e-6 * np.abs(want)), name
    np.testing.assert_array_equal(st.download(0, "pair_step"), orc.pair_step)
    comp = st.tensor(0, "w_a_compute").float().cpu().numpy()  # bf16 copy tracks the fp32 master
    master = st.download(0, "w_a").T
    assert np.all(np.abs(comp - master) <= np.abs(master) * 2.0 ** -8)


def test_device_checkpoint_matches_reference_bytes(ctx, tmp_path):
    """An F64 HBM store holding the reference store's state writes the reference's MEFT1 file byte for byte
    (memtier.cpp:288-326), router state included."""
    d, r, n = 16, 32, 4
    ref = O.RefStore(1, d, r, n, seed=5, train_router=True)
    rng = np.random.default_rng(3)
    for _ in range(2):
        s = np.sort(rng.choice(r, 6, replace=False))
        ref.scatter_grads(0, s, rng.standard_normal((d, 6)), rng.standard_normal((6, d)))
        ref.sparse_adam(0, 1e-2)
    ref.save(tmp_path / "ref.meft", extra='{"a": 1}', step=9)
    st = G.Store(ctx, 1, d, r, n, G.STORE_F64)
    st.enable_router()
    for name in ("w_a", "w_b", "w_g", "m_a", "v_a", "m_b", "v_b"):
        st.upload(0, name, ref.get(0, name))
    st.upload(0, "pair_step", ref.pair_step(0))
    # the reference's router moments are zero here (its STE lives in the trainer), counters too
    st.save(tmp_path / "dev.meft", step=9, extra='{"a": 1}')
    assert (tmp_path / "dev.meft").read_bytes() == (tmp_path / "ref.meft").read_bytes()


def test_mixed_store_checkpoint_resumes_bit_exactly(ctx, tmp_path):
    """save -> load of a trained MIXED store restores masters, moments, counters and compute copies exactly, and
    the next layer step of the resumed store equals the original's bit for bit."""
    d, M, N, T = 512, 4096, 64, 128
    st = G.Store(ctx, 1, d, M, N, G.STORE_MIXED)
    st.init_reference(seed=1)
    gen = torch.Generator(device="cuda").manual_seed(2)
    h = (torch.rand((T, d), generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16)
    g = (torch.rand((T, d), generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16)
    for _ in range(2):
        st.layer_step(0, h, g, 4, 32, 1e-3)
    st.save(tmp_path / "m.meft", step=2)
    st2, hdr, extra = G.Store.load(ctx, tmp_path / "m.meft", G.STORE_MIXED)
    assert (hdr.layers, hdr.dim, hdr.pairs, hdr.experts, hdr.step) == (1, d, M, N, 2) and extra == "{}"
    for name in ("w_a", "w_b", "w_g", "m_a", "v_a", "m_b", "v_b", "pair_step", "w_a_compute", "w_b_compute"):
        assert torch.equal(st.tensor(0, name), st2.tensor(0, name)), name
    outs = []
    for s_ in (st, st2):
        o = torch.empty((T, d), dtype=torch.float32, device="cuda")
        s_.layer_step(0, h, g, 4, 32, 1e-3, out=o)
        outs.append((o, s_.tensor(0, "w_b").clone()))
    torch.cuda.synchronize()
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("prec", ["f64", "mixed"])
def test_scatter_grads_repeated_ids_segmented_equals_sequential(ctx, prec):
    """scatter_grads with unsorted, heavily repeated neuron ids (memtier.cpp:139-149 adds entry by entry): the
    atomic-free segmented scatter (stable sort by id, one CTA per run) must equal the sequential loop bit for bit,
    and mark exactly the touched pairs as staged."""
    d, r, n = 40, 64, 500
    rs = np.random.RandomState(5)
    idx = rs.randint(0, 20, n).astype(np.int32)  # 500 entries on 20 pairs
    gk = rs.standard_normal((n, d))
    gv = rs.standard_normal((n, d))
    st = G.Store(ctx, 1, d, r, 4, G.STORE_F64 if prec == "f64" else G.STORE_MIXED)
    dt = torch.float64 if prec == "f64" else torch.float32
    st.scatter_grads(0, torch.from_numpy(idx).cuda(), torch.from_numpy(gk).to(dt).cuda(),
                     torch.from_numpy(gv).to(dt).cuda())
    cast = (lambda x: x) if prec == "f64" else (lambda x: x.astype(np.float32))
    want_a = np.zeros((r, d), dtype=np.float64 if prec == "f64" else np.float32)
    want_b = np.zeros_like(want_a)
    for j in range(n):  # the reference order: entry by entry
        want_a[idx[j]] = want_a[idx[j]] + cast(gk[j])
        want_b[idx[j]] = want_b[idx[j]] + cast(gv[j])
    np.testing.assert_array_equal(st.download(0, "stage_a").T.astype(want_a.dtype), want_a)
    np.testing.assert_array_equal(st.download(0, "stage_b").astype(want_b.dtype), want_b)
    staged = np.zeros(r, np.int8)
    staged[np.unique(idx)] = 1
    np.testing.assert_array_equal(st.download(0, "staged"), staged)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_rows_add_repeated_indices_equals_sequential_loop(ctx, dtype):
    """meft_rows_add (the drop-in's touched-row staging: scatter_grads / stage_router_grads on the mirrored rows):
    table[idx[i]] += rows[i] in entry order, flags[idx[i]] = 1 -- bit-identical to the reference's sequential loop
    (memtier.cpp:139-149) with repeated indices, and via the one-CTA-per-row path for strictly ascending ones."""
    import ctypes as C

    from paper_2406_04984_b200 import _lib

    gen = torch.Generator(device="cuda").manual_seed(4)
    n_rows, d = 37, 96
    for idx_list in ([3, 5, 5, 0, 36, 3, 3, 12], [0, 2, 7, 9, 30]):
        table = torch.randn((n_rows, d), generator=gen, device="cuda").to(dtype)
        rows = torch.randn((len(idx_list), d), generator=gen, device="cuda").to(dtype)
        idx = torch.tensor(idx_list, dtype=torch.int32, device="cuda")
        flags = torch.zeros(n_rows, dtype=torch.uint8, device="cuda")
        want = table.cpu().clone()
        for i, j in enumerate(idx_list):  # the reference's sequential loop
            want[j] += rows[i].cpu()
        dt = _lib.F64 if dtype == torch.float64 else _lib.F32
        ctx.check(_lib.lib().meft_rows_add(ctx.h, dt, C.c_void_p(table.data_ptr()), d, C.c_void_p(idx.data_ptr()),
                                           len(idx_list), C.c_void_p(rows.data_ptr()), C.c_void_p(flags.data_ptr())))
        torch.cuda.synchronize()
        assert torch.equal(table.cpu(), want)
        assert sorted(set(idx_list)) == torch.nonzero(flags).flatten().tolist()
