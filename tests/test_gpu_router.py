"""Trainable router on the fused layer step (train_router): the straight-through router gradient
(trainer.cpp:140-181, restated by oracle or_router_ste) staged and applied by the REFERENCE's own
stage_router_grads + sparse_adam_update (memtier.cpp:157-172, 211-227), against meft_layer_step on B200."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2406_04984_b200 import meft as G

pytestmark = pytest.mark.gpu


def bf16(x):
    return torch.from_numpy(np.ascontiguousarray(x)).float().to(torch.bfloat16)


def test_router_ste_and_adam_match_reference(ctx):
    d, M, N, K, T, kk, lr = 512, 4096, 64, 32, 256, 4, 1e-2
    E = M // N
    b = 1.0 / np.sqrt(d)
    w_a = O.bf16_round(O.uniform(O.mix_seed(1, 0x5000), (d, M), -b, b))
    w_g = O.bf16_round(O.uniform(O.mix_seed(1, 0x5001), (N, d), -b, b))
    w_b = O.bf16_round(O.uniform(O.mix_seed(1, 0x7001), (M, d), -b, b))
    h = O.bf16_round(O.uniform(O.mix_seed(1, 0x7002), (T, d), -1, 1))
    g = O.bf16_round(O.uniform(O.mix_seed(1, 0x7003), (T, d), -1, 1))

    # oracle: selection, forward z on the union, straight-through gradient
    sel = O.ke_select(h, w_g, w_a, kk, K)
    S = sel["unioned"]
    _, z, _ = O.ffn_forward(h, w_a[:, S], w_b[S, :])
    grad_g, touched = O.router_ste(h, z, w_b[S, :], S, sel["tau"], g, E, N)
    assert touched.sum() > N // 2
    # the reference applies it: stage_router_grads + the router rows of sparse_adam_update
    ref = O.RefStore(1, d, M, N, seed=1, train_router=True)
    ref.set(0, "w_g", w_g)
    rows = np.nonzero(touched)[0]
    ref.stage_router_grads(0, rows, grad_g[rows])
    ref.sparse_adam(0, lr)
    w_g_ref, m_g_ref, _, step_ref = ref.router(0)

    # GPU: the fused step with router training
    st = G.Store(ctx, 1, d, M, N, G.STORE_MIXED)
    st.enable_router()
    for name, v in (("w_a", w_a), ("w_g", w_g), ("w_b", w_b)):
        st.upload(0, name, v)
    res = st.layer_step(0, bf16(h).cuda(), bf16(g).cuda(), kk, K, lr, want_selection=True)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(res["unioned"].cpu().numpy(), S)
    np.testing.assert_array_equal(st.download(0, "router_step"), step_ref)  # same touched experts, exactly
    # gradient (first Adam step: m = (1 - beta1) g) within the bf16 tolerance
    g_gpu = st.download(0, "m_g") / 0.1
    assert np.linalg.norm(g_gpu - grad_g) / np.linalg.norm(grad_g) < 1e-2
    np.testing.assert_allclose(st.download(0, "m_g")[~touched], 0.0)
    # updated router weights: |dw_gpu - dw_ref| <= 1e-2 lr + 1e-6 |w|, sign-ambiguous entries up to 2 lr
    wg_gpu = st.download(0, "w_g")
    err = np.abs((wg_gpu - w_g) - (w_g_ref - w_g))
    assert np.all(err <= 2 * lr + 1e-6)
    strict = err <= 1e-2 * lr + 1e-6 * np.abs(w_g_ref)
    assert strict.mean() > 0.99, strict.mean()
    # the bf16 router copy the next selection reads follows the master
    assert torch.equal(st.tensor(0, "w_g_compute"), st.tensor(0, "w_g").to(torch.bfloat16))


def test_router_training_off_leaves_router_untouched(ctx):
    d, M, N, T = 512, 4096, 64, 128
    st = G.Store(ctx, 1, d, M, N, G.STORE_MIXED)
    st.init_reference(seed=1)
    w0 = st.tensor(0, "w_g").clone()
    h = (torch.rand((T, d), device="cuda") * 2 - 1).to(torch.bfloat16)
    st.layer_step(0, h, h, 4, 32, 1e-2)
    torch.cuda.synchronize()
    assert torch.equal(st.tensor(0, "w_g"), w0)


def test_trained_router_state_survives_checkpoint(ctx, tmp_path):
    d, M, N, T = 512, 4096, 64, 128
    st = G.Store(ctx, 1, d, M, N, G.STORE_MIXED)
    st.init_reference(seed=1)
    st.enable_router()
    gen = torch.Generator(device="cuda").manual_seed(4)
    h = (torch.rand((T, d), generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16)
    g = (torch.rand((T, d), generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16)
    for _ in range(2):
        st.layer_step(0, h, g, 4, 32, 1e-2)
    st.save(tmp_path / "r.meft", step=2)
    st2, hdr, _ = G.Store.load(ctx, tmp_path / "r.meft", G.STORE_MIXED)
    assert hdr.train_router == 1
    for name in ("w_g", "m_g", "v_g", "router_step", "w_g_compute"):
        a = st.tensor(0, name) if name not in ("m_g", "v_g", "router_step") else torch.from_numpy(st.download(0, name))
        b = st2.tensor(0, name) if name not in ("m_g", "v_g", "router_step") else torch.from_numpy(st2.download(0, name))
        assert torch.equal(a, b), name
    assert int(st2.download(0, "router_step").max()) == 2
