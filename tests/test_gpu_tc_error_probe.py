"""Directed probe of the tcgen05 accumulation error the certified selection relies on (select_tc.cuh:1-16).

The certificate assumes: each K=16 tcgen05 step adds 16 exact bf16 x bf16 products to the fp32 TMEM accumulator
with error at most 32 * 2^-24 * (|acc| + sum|p|) (CB(d) = 32 * 2^-24 * (ceil(d/16) + 1) + d * 2^-52). Random data
only samples that error statistically; here the scoring GEMM the selection uses (meft_score_candidates: grouped
tcgen05 GEMM, fp32 accumulation, no K split at d <= 1024) runs on ADVERSARIAL dot products built to maximise it:

  * align   : per 16-group one product of 1.0 and fifteen just under half an fp32 ulp of it (alignment shifts
              every small addend out of the accumulator's precision)
  * carry   : fifteen products of 2^-24 * (1 + j/128) after a large accumulator (rounding of the group sum)
  * cancel  : +A, -A pairs inside a group plus small terms of both signs (catastrophic cancellation, sum|p| >> |sum|)
  * ladder  : exponents stepping down 2^0 .. 2^-15 inside each group (every alignment distance at once)
  * spread  : random signs and exponents over [-24, 0]
  * random  : the uniform bf16 inputs of the bench

  * subulpK : an accumulator of 2^8, then every group's 16 products just under 2^-K ulp(acc) (K = 0..2): each addend
              lies below the accumulator's last bit, the worst case of an adder that aligns and truncates

For each dot the observed error |s_tc - x| (x = the exact sum, math.fsum of exact fp64 products) is expressed in
units of 2^-24 * sum_steps(|acc_before| + sum|p_step|): the model allows 32 units (16 ulp of |acc| per step). The
test asserts the model with a margin (at most half of it) for every family; the random-data families must stay
within 1/8 of it. The observed maxima per family are printed (DESIGN.md §3 records them)."""
import math

import numpy as np
import pytest
import torch

from paper_2406_04984_b200 import meft as G
from paper_2406_04984_b200 import sharded as SH

pytestmark = pytest.mark.gpu

MODEL_UNITS = 32.0


def bf16(x):
    f = np.ascontiguousarray(x, np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def family_rows(name, R, d, rng):
    """R rows of products p (R x d, every value bf16) for one adversarial family (keys are all ones)."""
    p = np.zeros((R, d))
    g = d // 16
    if name == "align":
        for s in range(g):
            p[:, 16 * s] = 1.0
            p[:, 16 * s + 1:16 * s + 16] = 2.0 ** -25 * (1.0 + rng.integers(0, 127, (R, 15)) / 128.0)
    elif name == "carry":
        p[:, 0] = 2.0 ** 8
        for s in range(1, g):
            p[:, 16 * s:16 * s + 16] = 2.0 ** -16 * (1.0 + rng.integers(0, 127, (R, 16)) / 128.0)
    elif name.startswith("subulp"):  # acc = 2^8, then 16 products per group just under 2^-k ulp(acc) each:
        k = int(name[-1])          # every addend sits below the accumulator's last bit (the truncation worst case)
        p[:, 0] = 2.0 ** 8
        for s in range(1, g):
            p[:, 16 * s:16 * s + 16] = (2.0 - 2.0 ** -7) * 2.0 ** (-16 - k)
    elif name == "cancel":
        for s in range(g):
            a = 2.0 ** rng.integers(-2, 3, R)
            p[:, 16 * s] = a
            p[:, 16 * s + 1] = -a
            p[:, 16 * s + 2:16 * s + 16] = (rng.choice([-1.0, 1.0], (R, 14)) * 2.0 ** rng.integers(-30, -20, (R, 14))
                                            * (1.0 + rng.integers(0, 127, (R, 14)) / 128.0))
    elif name == "ladder":
        for s in range(g):
            p[:, 16 * s:16 * s + 16] = (rng.choice([-1.0, 1.0], (R, 16)) * 2.0 ** -np.arange(16)
                                        * (1.0 + rng.integers(0, 127, (R, 16)) / 128.0))
    elif name == "spread":
        p = rng.choice([-1.0, 1.0], (R, d)) * 2.0 ** rng.integers(-24, 1, (R, d)) * (
            1.0 + rng.integers(0, 127, (R, d)) / 128.0)
    else:
        raise ValueError(name)
    return bf16(p)


def units(x_row, key, s):
    """(|s - exact|, model scale 2^-24 * sum_steps(|acc_before| + sum|p_step|)) of one dot."""
    p = x_row * key
    exact = math.fsum(p)
    scale, acc = 0.0, 0.0
    for s0 in range(0, len(p), 16):
        blk = p[s0:s0 + 16]
        scale += abs(acc) + float(np.abs(blk).sum())
        acc = math.fsum(p[:s0 + 16])
    return abs(float(s) - exact), scale * 2.0 ** -24


def score(ctx, rows, keys):
    """meft_score_candidates: every row against every key (one expert holding all keys), fp32 tcgen05 output."""
    R, d = rows.shape
    E = keys.shape[0]
    st = G.Store(ctx, 1, d, E, 1, G.STORE_MIXED)
    st.upload(0, "w_a", np.ascontiguousarray(keys.T))  # reference layout d x r; compute copy = bf16(keys) exactly
    eng = SH.DeviceEngine(ctx, st, st.tensor(0, "w_g_compute"))
    r = torch.from_numpy(rows).to(device="cuda", dtype=torch.bfloat16)
    cand = eng.score(r, torch.zeros(R, dtype=torch.int32, device="cuda"))
    torch.cuda.synchronize()
    out = cand.double().cpu().numpy()
    st.close()
    return out


@pytest.mark.parametrize("d", [256, 1024])
def test_tcgen05_accumulation_error_within_an_eighth_of_the_certificate_model(ctx, d):
    rng = np.random.default_rng(20 + d)
    R, E = 64, 8
    worst = {}
    for fam in ("align", "carry", "cancel", "ladder", "spread", "random", "subulp0", "subulp1", "subulp2"):
        if fam == "random":
            rows = bf16(rng.uniform(-1, 1, (R, d)))
            keys = bf16(rng.uniform(-1, 1, (E, d)) / math.sqrt(d))
        else:
            rows = family_rows(fam, R, d, rng)
            keys = np.ones((E, d))
            keys[1::2] = bf16(np.where(rng.random((E // 2, d)) < 0.5, 1.0, -1.0))  # sign flips keep products bf16
        s = score(ctx, rows, keys)
        w = 0.0
        for i in range(R):
            for j in range(E):
                err, sc = units(rows[i], keys[j], s[i, j])
                if sc > 0:
                    w = max(w, err / sc)
        worst[fam] = w
    print(f"\nd={d}: worst observed error in units of 2^-24*sum(|acc|+sum|p|): "
          + ", ".join(f"{k} {v:.3f}" for k, v in worst.items()) + f" (model {MODEL_UNITS:.0f})")
    assert max(worst.values()) <= MODEL_UNITS / 2
    assert max(worst[f] for f in ("spread", "random")) <= MODEL_UNITS / 8
