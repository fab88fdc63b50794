"""COMPACT stores (include/meft_cuda.h MEFT_STORE_COMPACT): MIXED with the Adam moments m, v kept in bf16, the
opt-in that fits BASELINE config 3 (32 LLaMA-7B-width layers) on one B200.

Stated tolerance: the Adam update itself runs in fp32 exactly as in MIXED, only the stored moments
are rounded to bf16 (relative 2^-9). Hence, against the MIXED store on the same inputs:
  * step 1: selection, out, grad_h and the updated weights are bit-identical (the first update uses the fresh fp32
    moments); m, v agree to within one bf16 rounding (relative 2^-8 entrywise)
  * step 2: selection identical (it reads the bf16 compute copies of the identical step-1 weights), and
    |w_compact - w_mixed| <= 2 * 2^-7 * lr entrywise (the second update's m/sqrt(v) carries <= ~2^-8 relative error)
  (later steps: the compute copies of weights that differ by ~1e-9 round differently in a handful of entries, so
  selections may legitimately diverge at near-ties; the per-step weight bound keeps holding for common pairs)
and the store's footprint is 20 B per (pair, dim) of tables instead of 28."""
import numpy as np
import pytest
import torch

from paper_2406_04984_b200 import meft as G

pytestmark = pytest.mark.gpu


def _pair(ctx, d, M, N, seed):
    stores = {}
    for name, prec in (("mixed", G.STORE_MIXED), ("compact", G.STORE_COMPACT)):
        st = G.Store(ctx, 1, d, M, N, prec)
        b = 1.0 / d ** 0.5
        st.upload(0, "w_a", G.reference_uniform(seed, 0x5000, (d, M), -b, b, bf16=True))
        st.upload(0, "w_g", G.reference_uniform(seed, 0x5001, (N, d), -b, b, bf16=True))
        st.upload(0, "w_b", G.reference_uniform(seed, 0x7001, (M, d), -b, b, bf16=True))
        stores[name] = st
    return stores


@pytest.mark.parametrize("shape", [(512, 4096, 64, 32, 256), (1024, 16384, 64, 64, 2048)])
def test_compact_moments_track_mixed_within_stated_tolerance(ctx, shape):
    d, M, N, K, T = shape
    kk, lr, steps = 4, 1e-3, 2
    st = _pair(ctx, d, M, N, 7)
    assert st["compact"].precision == G.STORE_COMPACT
    assert st["compact"].tensor(0, "m_a").dtype == torch.bfloat16 and st["mixed"].tensor(0, "m_a").dtype == torch.float32
    res = {}
    for step in range(1, steps + 1):
        h = torch.from_numpy(G.reference_uniform(3, 0x7002 + step, (T, d), -1, 1, bf16=True)).cuda().bfloat16()
        g = torch.from_numpy(G.reference_uniform(3, 0x7003 + step, (T, d), -1, 1, bf16=True)).cuda().bfloat16()
        for name, s in st.items():
            out = torch.empty((T, d), device="cuda")
            gh = torch.empty_like(out)
            r = s.layer_step(0, h, g, kk, K, lr, out=out, grad_h=gh, want_selection=True)
            res[name] = (r, out, gh)
        torch.cuda.synchronize()
        rm, rc = res["mixed"][0], res["compact"][0]
        assert torch.equal(rm["per_token"], rc["per_token"]) and torch.equal(rm["unioned"], rc["unioned"])
        if step == 1:
            assert torch.equal(res["mixed"][1], res["compact"][1]) and torch.equal(res["mixed"][2], res["compact"][2])
        for tab in ("a", "b"):
            wm, wc = st["mixed"].tensor(0, "w_" + tab), st["compact"].tensor(0, "w_" + tab)
            dw = (wm - wc).abs().max().item()
            if step == 1:
                assert dw == 0.0, (tab, dw)
            assert dw <= step * 2.0 ** -7 * lr + 1e-9, (step, tab, dw, lr)
            for mom in ("m", "v"):
                xm = st["mixed"].tensor(0, f"{mom}_{tab}")
                xc = st["compact"].tensor(0, f"{mom}_{tab}").float()
                if step == 1:  # one rounding of the same fp32 value
                    assert torch.all((xc - xm).abs() <= xm.abs() * 2.0 ** -8), (mom, tab)
                rel = ((xc - xm).norm() / xm.norm()).item()
                assert rel < 2.0 ** -7 * step, (step, mom, tab, rel)


def test_compact_store_footprint_and_checkpoint_round_trip(ctx, tmp_path):
    d, M, N = 256, 2048, 16
    free0 = torch.cuda.mem_get_info()[0]
    st = G.Store(ctx, 2, d, M, N, G.STORE_COMPACT)
    used = free0 - torch.cuda.mem_get_info()[0]
    assert used <= 2 * (M * d * 20 + (2 << 20)) + (4 << 20), used  # 20 B per (pair, dim) + small per-layer tables
    b = 1.0 / d ** 0.5
    st.upload(0, "w_a", G.reference_uniform(1, 0x5000, (d, M), -b, b, bf16=True))
    st.upload(0, "w_b", G.reference_uniform(1, 0x7001, (M, d), -b, b, bf16=True))
    st.upload(0, "w_g", G.reference_uniform(1, 0x5001, (N, d), -b, b, bf16=True))
    h = torch.from_numpy(G.reference_uniform(1, 0x7002, (64, d), -1, 1, bf16=True)).cuda().bfloat16()
    st.layer_step(0, h, h, 4, 16, 1e-3)
    torch.cuda.synchronize()
    path = tmp_path / "c.meft"
    st.save(path, step=5)
    back, hdr, _ = G.Store.load(ctx, path, G.STORE_COMPACT)
    assert hdr.step == 5
    for name in ("w_a", "w_b", "m_a", "v_a", "m_b", "v_b", "pair_step"):
        a, c = st.download(0, name), back.download(0, name)
        assert np.array_equal(a, c), name  # bf16 moments are exact in the file's f64
    back.close()
    st.close()
