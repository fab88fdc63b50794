"""GPU parity of the sparse FFN forward/backward (adapter.cpp:112-180).

float64 path (API fidelity): bitwise / 1e-13 against the oracle (same ascending-k fma chains).
bf16 tcgen05 path: normwise relative error <= 1e-2 against the fp64 oracle on bf16-rounded inputs
(bf16 operands, fp32 TMEM accumulation, bf16 ReLU(z) / masked intermediates)."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2406_04984_b200 import meft as G

pytestmark = pytest.mark.gpu

BF16_TOL = 1e-2


def dev(x, dtype):
    t = torch.from_numpy(np.ascontiguousarray(x))
    return (t.float().to(torch.bfloat16) if dtype == "bf16" else t.double()).cuda().contiguous()


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def test_f64_matches_reference_fixture(ctx, golden):
    g = golden("ffn.npz")
    for i in range(int(g["n"])):
        c = lambda k: g[f"c{i}__{k}"]  # noqa: E731
        if c("w_in").shape[1] != 0:
            continue  # adapter half only here; the base half is covered by the drop-in tests
        h, wak, wbk = c("h"), c("w_a")[:, c("S")], c("w_b")[c("S"), :]
        z, out, ld = G.ffn_forward(ctx, dev(h, "f64"), dev(wak.T, "f64"), dev(wbk, "f64"))
        np.testing.assert_array_equal(z.cpu().numpy()[:, : wak.shape[1]], c("z"))
        np.testing.assert_allclose(out.cpu().numpy(), c("out"), rtol=1e-13, atol=1e-14)
        gk, gv, gh = G.ffn_backward(ctx, dev(c("G"), "f64"), dev(h, "f64"), z, dev(wak.T, "f64"), dev(wbk, "f64"), ld)
        np.testing.assert_allclose(gk.cpu().numpy().T, c("gwa"), rtol=1e-13, atol=1e-14)
        np.testing.assert_allclose(gv.cpu().numpy(), c("gwb"), rtol=1e-13, atol=1e-14)
        np.testing.assert_allclose(gh.cpu().numpy(), c("gh"), rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("T,d,s", [(1, 8, 1), (3, 16, 5), (37, 64, 100), (130, 96, 257)])
def test_f64_random_vs_oracle_bitwise(ctx, T, d, s):
    h, wak, wbk, Gm = (O.uniform(T * 7 + i, shp, -1, 1) for i, shp in enumerate([(T, d), (d, s), (s, d), (T, d)]))
    out_o, z_o, _ = O.ffn_forward(h, wak, wbk)
    gwa_o, gwb_o, gh_o = O.ffn_backward(Gm, h, z_o, None, wak, wbk)
    z, out, ld = G.ffn_forward(ctx, dev(h, "f64"), dev(wak.T, "f64"), dev(wbk, "f64"))
    gk, gv, gh = G.ffn_backward(ctx, dev(Gm, "f64"), dev(h, "f64"), z, dev(wak.T, "f64"), dev(wbk, "f64"), ld)
    np.testing.assert_array_equal(z.cpu().numpy(), z_o)
    np.testing.assert_array_equal(out.cpu().numpy(), out_o)
    np.testing.assert_array_equal(gv.cpu().numpy(), gwb_o)
    np.testing.assert_allclose(gk.cpu().numpy().T, gwa_o, rtol=1e-14, atol=1e-15)
    np.testing.assert_array_equal(gh.cpu().numpy(), gh_o)


@pytest.mark.parametrize("T,d,s", [(128, 64, 256), (256, 512, 3487), (200, 136, 333), (64, 4096, 1000)])
def test_bf16_tcgen05_vs_fp64_oracle(ctx, T, d, s):
    bound = 1.0 / np.sqrt(d)
    h = O.bf16_round(O.uniform(1, (T, d), -1, 1))
    wak = O.bf16_round(O.uniform(2, (d, s), -bound, bound))
    wbk = O.bf16_round(O.uniform(3, (s, d), -bound, bound))
    Gm = O.bf16_round(O.uniform(4, (T, d), -1, 1))
    out_o, z_o, _ = O.ffn_forward(h, wak, wbk)
    gwa_o, gwb_o, gh_o = O.ffn_backward(Gm, h, z_o, None, wak, wbk)
    act, out, ld = G.ffn_forward(ctx, dev(h, "bf16"), dev(wak.T, "bf16"), dev(wbk, "bf16"))
    gk, gv, gh = G.ffn_backward(ctx, dev(Gm, "bf16"), dev(h, "bf16"), act, dev(wak.T, "bf16"), dev(wbk, "bf16"), ld)
    torch.cuda.synchronize()
    a = act[:, :s].float().cpu().numpy()
    np.testing.assert_allclose(a, np.maximum(z_o, 0), rtol=1e-2, atol=1e-5 * np.abs(z_o).max())
    # the ReLU mask may differ from fp64 only where |z| is below the fp32 accumulation error
    flip = (a > 0) != (z_o > 0)
    assert np.all(np.abs(z_o[flip]) < 1e-4 * np.abs(z_o).max())
    assert rel(out.cpu().numpy(), out_o) < BF16_TOL
    assert rel(gv.cpu().numpy(), gwb_o) < BF16_TOL
    assert rel(gk.cpu().numpy().T, gwa_o) < BF16_TOL
    assert rel(gh.cpu().numpy(), gh_o) < BF16_TOL


def test_empty_selection(ctx):
    h = dev(O.uniform(1, (4, 8), -1, 1), "f64")
    e = torch.zeros((0, 8), dtype=torch.float64, device="cuda")
    z, out, ld = G.ffn_forward(ctx, h, e, e)
    assert float(out.abs().max()) == 0.0  # sparse_ffn_pa with empty S == base only (test_adapter.cpp:187-193)
    gk, gv, gh = G.ffn_backward(ctx, h, h, z, e, e, ld)
    assert gk.shape == (0, 8) and float(gh.abs().max()) == 0.0


def test_no_firing_kills_adapter_grads(ctx):  # test_adapter.cpp:232-247
    h = np.abs(O.uniform(5, (2, 8), -1, 1)) + 0.5
    wak = -2.0 - np.abs(O.uniform(6, (8, 5), -1, 1))
    wbk = O.uniform(7, (5, 8), -1, 1)
    z, out, ld = G.ffn_forward(ctx, dev(h, "f64"), dev(wak.T, "f64"), dev(wbk, "f64"))
    assert float(z.max()) < 0
    gk, gv, gh = G.ffn_backward(ctx, dev(O.uniform(8, (2, 8), -1, 1), "f64"), dev(h, "f64"), z, dev(wak.T, "f64"),
                                dev(wbk, "f64"), ld)
    assert float(gk.abs().max()) == 0.0 and float(gv.abs().max()) == 0.0


def test_gather_adapter_validation(ctx):
    keys = dev(O.uniform(8, (4, 3), -1, 1), "f64")
    vals = dev(O.uniform(9, (4, 3), -1, 1), "f64")
    ks, vs = G.gather_adapter(ctx, keys, vals, torch.tensor([0, 2, 3], dtype=torch.int32, device="cuda"))
    np.testing.assert_array_equal(ks.cpu().numpy(), keys.cpu().numpy()[[0, 2, 3]])
    with pytest.raises(G.MeftError) as e:
        G.gather_adapter(ctx, keys, vals, torch.tensor([2, 0], dtype=torch.int32, device="cuda"))
    assert e.value.kind == "invalid_argument"
    with pytest.raises(G.MeftError) as e:
        G.gather_adapter(ctx, keys, vals, torch.tensor([7], dtype=torch.int32, device="cuda"))
    assert e.value.kind == "out_of_range" and e.value.index == 7 and "7" in str(e.value)
