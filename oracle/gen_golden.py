"""ORACLE / TEST INFRASTRUCTURE: regenerate tests/golden/*.npz from the UNMODIFIED reference.

Runs only where /root/reference exists (this build container): it compiles oracle/_ref/libmeft_ref.so via
oracle/Makefile and records, for seeded inputs, what the reference's public API returns. Small cases store
their inputs verbatim; the cfg1-sized cases store the RNG seeds (the RNG itself is pinned by rng.npz) plus
input checksums. Usage:  python oracle/gen_golden.py
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def ref_uniform(seed, shape, lo, hi):
    r = O.ref()
    out = np.empty(int(np.prod(shape)))
    r.ref_uniform_matrix(O.C.c_uint64(seed), O._I64(shape[0]), O._I64(int(np.prod(shape[1:])) if len(shape) > 1 else 1),
                         O._D(lo), O._D(hi), O._ptr(out))
    return out.reshape(shape)


def gen_rng():
    seeds = [(1, 0x7001), (1, 0x7002), (99, 0x5002), (5, 0)]
    mixed = np.array([O.ref().ref_mix_seed(s, t) for s, t in seeds], dtype=np.uint64)
    draws = np.stack([ref_uniform(int(m), (64,), -0.5, 0.25) for m in mixed])
    np.savez_compressed(os.path.join(OUT, "rng.npz"), seeds=np.array(seeds, dtype=np.uint64), mixed=mixed,
                        draws=draws)


def selection_case(name, T, d, r, N, kk, k, seed, bf16):
    mk = lambda s, shape: O.uniform(O.mix_seed(seed, s), shape, -1.0, 1.0)  # noqa: E731
    h, w_a, w_g = mk(1, (T, d)), mk(2, (d, r)), mk(3, (N, d))
    if bf16:
        h, w_a, w_g = O.bf16_round(h), O.bf16_round(w_a), O.bf16_round(w_g)
    res = O.ref_ke_select(h, w_g, w_a, kk, k)
    flat = O.ref_topk_select(h, w_a, k)
    return dict(T=T, d=d, r=r, N=N, kk=kk, k=k, seed=seed, bf16=int(bf16), inputs_sha=digest(h, w_a, w_g),
                per_token=res["per_token"], tau=res["tau"], unioned=res["unioned"], take=res["take"],
                flat_per_token=flat["per_token"], flat_unioned=flat["unioned"])


def gen_selection():
    cases = {
        "cfg1_bf16": (256, 512, 4096, 64, 4, 32, 11, True),
        "cfg1_f64": (64, 512, 4096, 64, 4, 32, 12, False),
        "odd_d_f64": (40, 33, 96, 8, 3, 7, 13, False),
        "clamp": (8, 16, 64, 8, 1, 20, 14, False),
        "full_budget": (12, 8, 48, 4, 4, 5, 15, False),
        "one_expert": (12, 8, 48, 1, 1, 5, 16, True),
    }
    out = {}
    for name, args in cases.items():
        for key, v in selection_case(name, *args).items():
            out[f"{name}__{key}"] = v
    np.savez_compressed(os.path.join(OUT, "selection.npz"), names=np.array(list(cases)), **out)


def gen_ffn():
    rng_seed = 21
    out = {}
    configs = [(3, 4, 5, 6, 0), (6, 8, 10, 16, 1), (5, 7, 0, 9, 0), (4, 16, 12, 32, 1)]  # (T, d, n, r, act)
    for i, (T, d, n, r, act) in enumerate(configs):
        mk = lambda s, shape: O.uniform(O.mix_seed(rng_seed + i, s), shape, -1.0, 1.0)  # noqa: E731
        h, w_in, w_out, w_a, w_b, G = mk(1, (T, d)), mk(2, (d, n)), mk(3, (n, d)), mk(4, (d, r)), mk(5, (r, d)), mk(6, (T, d))
        sel = O.ref_topk_select(h, w_a, max(1, r // 3))["unioned"]
        wak, wbk = w_a[:, sel], w_b[sel, :]
        y, z, pre = O.ref_ffn_forward(h, wak, wbk, w_in if n else None, w_out if n else None, act)
        gwa, gwb, gh = O.ref_ffn_backward(h, wak, wbk, G, w_in if n else None, w_out if n else None, act)
        for key, v in dict(h=h, w_in=w_in, w_out=w_out, w_a=w_a, w_b=w_b, G=G, S=sel, out=y, z=z, base_pre=pre,
                           gwa=gwa, gwb=gwb, gh=gh, act=act).items():
            out[f"c{i}__{key}"] = v
    np.savez_compressed(os.path.join(OUT, "ffn.npz"), n=len(configs), **out)


def gen_adam():
    """Three scatter+Adam steps on a small reference store (memtier.cpp:128-228)."""
    L, d, r, N = 2, 3, 6, 2
    st = O.RefStore(L, d, r, N, seed=99)
    out = dict(w_a0=st.get(0, "w_a"), w_b0=st.get(0, "w_b"), w_g0=st.get(0, "w_g"), w_a1=st.get(1, "w_a"))
    plans = [([1, 4], 1e-3), ([0, 4, 5], 5e-3), ([4], 1e-2)]
    for i, (S, lr) in enumerate(plans):
        ga = O.uniform(O.mix_seed(7, i), (d, len(S)), -1, 1)
        gb = O.uniform(O.mix_seed(8, i), (len(S), d), -1, 1)
        st.scatter_grads(0, S, ga, gb)
        st.sparse_adam(0, lr)
        out[f"s{i}__S"] = np.array(S)
        out[f"s{i}__lr"] = lr
        out[f"s{i}__ga"] = ga
        out[f"s{i}__gb"] = gb
        for name in ("w_a", "w_b", "m_a", "v_a", "m_b", "v_b"):
            out[f"s{i}__{name}"] = st.get(0, name)
        out[f"s{i}__pair_step"] = st.pair_step(0)
    np.savez_compressed(os.path.join(OUT, "adam.npz"), steps=len(plans), d=d, r=r, **out)


def gen_layer_step():
    """A full reference layer step at the cfg1 shape (d=512, M=4096, N=64, K=32, T=256) on bf16-rounded
    tables; stores checksums of the outputs, the selection and the updated tables (inputs by seed)."""
    d, M, N, K, T, kk, lr = 512, 4096, 64, 32, 256, 4, 1e-4
    st = O.RefStore(1, d, M, N, seed=1)
    bound = 1.0 / np.sqrt(d)
    w_a = O.bf16_round(st.get(0, "w_a"))
    w_g = O.bf16_round(st.get(0, "w_g"))
    w_b = O.bf16_round(O.uniform(O.mix_seed(1, 0x7001), (M, d), -bound, bound))
    h = O.bf16_round(O.uniform(O.mix_seed(1, 0x7002), (T, d), -1.0, 1.0))
    G = O.bf16_round(O.uniform(O.mix_seed(1, 0x7003), (T, d), -1.0, 1.0))
    st.set(0, "w_a", w_a)
    st.set(0, "w_g", w_g)
    st.set(0, "w_b", w_b)
    sel = O.ref_ke_select(h, w_g, w_a, kk, K)
    res = st.layer_step(0, h, G, kk, K, lr)
    toks = np.arange(0, T, 8)          # 32 sampled tokens of out / grad_h
    pairs = np.arange(0, M, 61)        # 68 sampled pairs of the updated tables
    w_a_after, w_b_after = st.get(0, "w_a"), st.get(0, "w_b")
    np.savez_compressed(os.path.join(OUT, "layer_cfg1.npz"), d=d, M=M, N=N, K=K, T=T, kk=kk, lr=lr,
                        per_token=sel["per_token"].astype(np.int16), tau=sel["tau"].astype(np.int16),
                        unioned=sel["unioned"].astype(np.int16), union_size=res["union_size"],
                        toks=toks, out=res["out"][toks], grad_h=res["grad_h"][toks],
                        out_fro=np.linalg.norm(res["out"]), grad_h_fro=np.linalg.norm(res["grad_h"]),
                        pairs=pairs, w_a_after=w_a_after[:, pairs], w_b_after=w_b_after[pairs, :],
                        pair_step=st.pair_step(0).astype(np.int8), inputs_sha=digest(w_a, w_g, w_b, h, G))


if __name__ == "__main__":
    O.build()
    if not O.ref_available():
        sys.exit("reference build unavailable (needs /root/reference)")
    os.makedirs(OUT, exist_ok=True)
    gen_rng()
    gen_selection()
    gen_ffn()
    gen_adam()
    gen_layer_step()
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))
