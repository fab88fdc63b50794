"""Value parity at the exact bench configuration (BASELINE.json configs[1], bench.py's workload): d=4096, M=65,536,
N=256, K=128, kk=4, T=8,192, bf16, one fused layer step on the B200 against the UNMODIFIED reference (oracle/_ref)
on the same inputs -- HostStore::init(seed 1) tables and the BASELINE.md §3 streams (W_B 0x7001, h 0x7002,
grad_out 0x7003), all bf16-rounded, so both sides score identical values.

  * indices: the per-token top-K and the union of ALL 8,192 tokens == the reference's ke_select (experts.cpp:47-117)
  * out / grad_h of 32 tokens spread over the batch == sparse_ffn_pa / sparse_backward of those rows against the
    whole union (adapter.cpp:112-180; rows are independent), normwise within the bf16 tolerance below
  * the Adam-updated rows of 64 pairs spread over the union (w, m, v of the key column and value row) == the
    reference's scatter_grads + sparse_adam_update (memtier.cpp:128-228) of those pairs' full-batch gradients

Tolerances are per tensor, about 2.5x the error observed on B200 (out 1.65e-3, grad_h 1.76e-3, gradients 1.65-1.72e-3,
v 1.9-2.0e-3; printed by the test), so an accuracy regression of 3x fails. The reference work is sized to run in well under a minute on 16 cores."""
import math

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2406_04984_b200 import meft as G

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

D, M, N, K, KK, T, LR = 4096, 65536, 256, 128, 4, 8192, 1e-4
# normwise relative error bounds vs the fp64 reference (observed on B200 x ~2.5)
TOL = {"out": 4.5e-3, "grad_h": 4.5e-3, "grad_w_a": 4.5e-3, "grad_w_b": 4.5e-3, "v_a": 5.5e-3, "v_b": 5.5e-3}
N_TOKENS, N_PAIRS = 32, 64


def rel(a, r):
    return float(np.linalg.norm(np.asarray(a, np.float64) - r) / np.linalg.norm(r))


@pytest.fixture(scope="module")
def step(ctx):
    if not O.ref_available():
        pytest.skip("oracle/_ref (the compiled reference) is not built")
    b = 1.0 / math.sqrt(D)
    w_a = G.reference_uniform(1, 0x5000, (D, M), -b, b, bf16=True)  # HostStore::init stream of layer 0
    w_g = G.reference_uniform(1, 0x5001, (N, D), -b, b, bf16=True)
    w_b = G.reference_uniform(1, 0x7001, (M, D), -b, b, bf16=True)
    h = G.reference_uniform(1, 0x7002, (T, D), -1.0, 1.0, bf16=True)
    g = G.reference_uniform(1, 0x7003, (T, D), -1.0, 1.0, bf16=True)

    st = G.Store(ctx, 1, D, M, N, G.STORE_MIXED)
    st.upload(0, "w_a", w_a)
    st.upload(0, "w_g", w_g)
    st.upload(0, "w_b", w_b)
    bf = lambda x: torch.from_numpy(x).to(device="cuda", dtype=torch.bfloat16)  # noqa: E731 (exact: bf16 values)
    out = torch.empty((T, D), dtype=torch.float32, device="cuda")
    gh = torch.empty_like(out)
    res = st.layer_step(0, bf(h), bf(g), KK, K, LR, out=out, grad_h=gh, want_selection=True)
    torch.cuda.synchronize()
    gpu = dict(per_token=res["per_token"].cpu().numpy(), unioned=res["unioned"].cpu().numpy(),
               tau=res["tau"].cpu().numpy() if res.get("tau") is not None else None,
               out=out.cpu().numpy(), grad_h=gh.cpu().numpy())
    ref_sel = O.ref_ke_select(h, w_g, w_a, KK, K)
    S = ref_sel["unioned"]
    toks = np.linspace(0, T - 1, N_TOKENS).astype(np.int64)
    pairs = S[np.linspace(0, len(S) - 1, N_PAIRS).astype(np.int64)]
    pair_pos = np.searchsorted(S, pairs)
    tables = {name: st.tensor(0, name) for name in ("w_a", "m_a", "v_a", "w_b", "m_b", "v_b")}
    jj = torch.from_numpy(pairs).cuda()
    gpu.update({name: t[jj].double().cpu().numpy() for name, t in tables.items()})  # neuron-major rows
    gpu["pair_step"] = st.download(0, "pair_step")
    yield dict(w_a=w_a, w_b=w_b, w_g=w_g, h=h, g=g, gpu=gpu, ref_sel=ref_sel, toks=toks, pairs=pairs,
               pair_pos=pair_pos, res=res)
    st.close()


def test_indices_of_all_8192_tokens_equal_the_reference(step):
    gpu, ref = step["gpu"], step["ref_sel"]
    assert gpu["per_token"].shape == ref["per_token"].shape == (T, K)
    bad = np.nonzero((gpu["per_token"] != ref["per_token"]).any(1))[0]
    assert bad.size == 0, f"{bad.size} tokens differ, first {bad[:8].tolist()}"
    assert np.array_equal(gpu["unioned"], ref["unioned"])
    if gpu["tau"] is not None:
        assert np.array_equal(gpu["tau"], ref["tau"])
    print(f"\ncfg2 selection: all {T} tokens bit-exact, |S| = {len(ref['unioned'])}, rescored per token "
          f"{step['res'].get('rescored', 0) / T:.2f}")


def test_out_and_grad_h_of_sampled_tokens(step):
    S, toks = step["ref_sel"]["unioned"], step["toks"]
    w_a_k, w_b_k = step["w_a"][:, S], step["w_b"][S, :]
    h, g = step["h"][toks], step["g"][toks]
    out_ref, _, _ = O.ref_ffn_forward(h, w_a_k, w_b_k)
    _, _, gh_ref = O.ref_ffn_backward(h, w_a_k, w_b_k, g)
    e_out, e_gh = rel(step["gpu"]["out"][toks], out_ref), rel(step["gpu"]["grad_h"][toks], gh_ref)
    print(f"\ncfg2 {N_TOKENS} tokens: out normwise rel err {e_out:.3e} (tol {TOL['out']}), "
          f"grad_h {e_gh:.3e} (tol {TOL['grad_h']})")
    assert e_out < TOL["out"] and e_gh < TOL["grad_h"]
    # and row by row (no single token hides behind the norm)
    per_row = [rel(step["gpu"]["out"][t], o) for t, o in zip(toks, out_ref)]
    assert max(per_row) < 3 * TOL["out"], per_row


def test_adam_updated_rows_of_sampled_pairs(step):
    """The sampled pairs' full-batch gradients from the reference (sparse_backward restricted to those columns:
    each pair's gradient depends only on its own key column and value row), then the reference's own
    scatter_grads + sparse_adam_update on a store holding just those pairs."""
    pairs, gpu = step["pairs"], step["gpu"]
    w_a_j, w_b_j = step["w_a"][:, pairs], step["w_b"][pairs, :]
    gwa, gwb, _ = O.ref_ffn_backward(step["h"], w_a_j, w_b_j, step["g"])  # d x P, P x d
    rs = O.RefStore(1, D, N_PAIRS, 1, seed=1)
    rs.set(0, "w_a", w_a_j)
    rs.set(0, "w_b", w_b_j)
    rs.scatter_grads(0, np.arange(N_PAIRS), gwa, gwb)
    rs.sparse_adam(0, LR)
    ref = {name: rs.get(0, name) for name in ("w_a", "m_a", "v_a", "w_b", "m_b", "v_b")}
    assert np.array_equal(gpu["pair_step"][pairs], np.ones(N_PAIRS, np.int64))  # one step per touched pair
    errs = {}
    # m = (1 - b1) g after the first step: the gradient, normwise
    errs["grad_w_a"] = rel(gpu["m_a"], ref["m_a"].T)
    errs["grad_w_b"] = rel(gpu["m_b"], ref["m_b"])
    errs["v_a"] = rel(gpu["v_a"], ref["v_a"].T)
    errs["v_b"] = rel(gpu["v_b"], ref["v_b"])
    print("\ncfg2 64 pairs: " + ", ".join(f"{k} {v:.3e} (tol {TOL[k]})" for k, v in errs.items()))
    for k, v in errs.items():
        assert v < TOL[k], (k, v)
    # the weight step: |dw_gpu - dw_ref| <= 1e-2 lr + 1 ulp (fp32 master), except entries whose gradient sign is
    # not determined at bf16 precision (|g_ref| inside the gradient error band): those may move up to 2 lr
    for name, w0, g_ref in (("w_a", w_a_j.T, gwa.T), ("w_b", w_b_j, gwb)):
        w_ref = ref[name].T if name == "w_a" else ref[name]
        dw_gpu, dw_ref = gpu[name] - w0, w_ref - w0
        diff = np.abs(dw_gpu - dw_ref)
        band = 3 * errs["grad_" + name] * np.sqrt(np.mean(g_ref ** 2))  # per-entry gradient error scale
        ambiguous = np.abs(g_ref) <= band
        ok = diff <= 1e-2 * LR + np.spacing(np.abs(w0).astype(np.float32)).astype(np.float64)
        assert np.all(ok | ambiguous), (name, int((~ok & ~ambiguous).sum()))
        assert np.all(diff[ambiguous] <= 2 * LR + 1e-9)
        print(f"cfg2 {name}: max |dw_gpu - dw_ref| = {diff[~ambiguous].max():.2e} "
              f"(lr = {LR}), sign-ambiguous entries {int(ambiguous.sum())} of {ambiguous.size}")
