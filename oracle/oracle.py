"""ORACLE / TEST INFRASTRUCTURE ONLY.

numpy-facing ctypes wrappers over
  * ``_build/libmeft_oracle.so`` -- the C restatement (meft_oracle.c), and
  * ``_ref/libmeft_ref.so``      -- the UNMODIFIED reference compiled by oracle/Makefile.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline / ``--impl reference``
legs may import this module. The product path (paper_2406_04984_b200) never does.

Layouts are the reference's (proj/include/meft/adapter.hpp:20-26): ``w_a`` is d x r with keys
as columns, ``w_b`` r x d, ``w_g`` N x d, ``h`` T x d, float64; indices int64.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libmeft_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmeft_ref.so")

_P = C.c_void_p
_I64 = C.c_int64
_D = C.c_double


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_P)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


class OracleError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build()
        _lib = C.CDLL(ORACLE_SO)
        _lib.or_mix_seed.restype = C.c_uint64
        _lib.or_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        _lib.or_dot.restype = _D
        _lib.or_select_experts.restype = _I64
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        _ref = C.CDLL(REF_SO)
        _ref.ref_last_error.restype = C.c_char_p
        _ref.ref_mix_seed.restype = C.c_uint64
        _ref.ref_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        _ref.ref_store_init.restype = _P
        _ref.ref_store_init.argtypes = [_I64, _I64, _I64, _I64, C.c_int, C.c_uint64]
        _ref.ref_store_free.argtypes = [_P]
        _ref.ref_warn_count.restype = C.c_long
        _ref.ref_step_begin.restype = _P
        _ref.ref_step_begin.argtypes = [_P, _I64, _P, _I64, _I64, _I64, _P, _P, _P]
        _ref.ref_step_rows.argtypes = [_P, _P, _P, _I64, _P, _P]
        _ref.ref_step_finish.argtypes = [_P, _P, _D, _P, _P]
    return _ref


def _check_ref(code):
    if code != 0:
        raise OracleError(code, ref().ref_last_error().decode())


# ----------------------------------------------------------------- RNG (rng.hpp)

def mix_seed(seed: int, stream: int) -> int:
    return int(lib().or_mix_seed(seed, stream))


def uniform(seed: int, shape, lo: float, hi: float) -> np.ndarray:
    """SeededRng(seed).uniform_matrix(...) (rng.hpp:62-66), row-major."""
    n = int(np.prod(shape))
    out = np.empty(n, dtype=np.float64)
    lib().or_uniform_matrix(C.c_uint64(seed), _I64(n), _D(lo), _D(hi), _ptr(out))
    return out.reshape(shape)


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round float64 -> bf16 (RNE via float32) -> back to float64 exactly."""
    f = np.ascontiguousarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


# ------------------------------------------------------------ restatement (or_*)

def ke_select(h, w_g, w_a, kk, k):
    h, w_g, w_a = _f64(h), _f64(w_g), _f64(w_a)
    T, d = h.shape
    N = w_g.shape[0]
    r = w_a.shape[1]
    kk_eff = min(kk, N)
    cap = max(1, min(k, kk_eff * (r // max(N, 1))))
    per = np.empty((T, cap), np.int64)
    tau = np.empty((T, kk_eff), np.int64)
    uni = np.empty(r, np.int64)
    us, take, warned = _I64(), _I64(), C.c_int()
    code = lib().or_ke_select(_ptr(h), _I64(T), _I64(d), _ptr(w_g), _I64(N), _ptr(w_a), _I64(r), _I64(kk),
                              _I64(k), _ptr(per), _ptr(tau), _ptr(uni), C.byref(us), C.byref(take),
                              C.byref(warned))
    if code:
        raise OracleError(code)
    return dict(per_token=per[:, : take.value].copy(), tau=tau, unioned=uni[: us.value].copy(),
                take=take.value, warned=bool(warned.value))


def topk_select(h, w_a, k):
    h, w_a = _f64(h), _f64(w_a)
    T, d = h.shape
    r = w_a.shape[1]
    cap = max(1, min(k, r))
    per = np.empty((T, cap), np.int64)
    uni = np.empty(r, np.int64)
    us, take, warned = _I64(), _I64(), C.c_int()
    code = lib().or_topk_select(_ptr(h), _I64(T), _I64(d), _ptr(w_a), _I64(r), _I64(k), _ptr(per), _ptr(uni),
                                C.byref(us), C.byref(take), C.byref(warned))
    if code:
        raise OracleError(code)
    return dict(per_token=per[:, : take.value].copy(), unioned=uni[: us.value].copy(), take=take.value,
                warned=bool(warned.value))


def route_scores(h_token, w_g):
    h_token, w_g = _f64(h_token), _f64(w_g)
    p = np.empty(w_g.shape[0])
    lib().or_route_scores(_ptr(h_token), _I64(w_g.shape[1]), _ptr(w_g), _I64(w_g.shape[0]), _ptr(p))
    return p


def select_experts(p, kk):
    p = _f64(p)
    out = np.empty(max(1, len(p)), np.int64)
    take = lib().or_select_experts(_ptr(p), _I64(len(p)), _I64(kk), _ptr(out))
    if take < 0:
        raise OracleError(2, "select_experts: budget must be >= 1")
    return out[:take].copy()


def gather_adapter(w_a, w_b, s):
    w_a, w_b, s = _f64(w_a), _f64(w_b), _i64(s)
    d, r = w_a.shape
    wak = np.empty((d, len(s)))
    wbk = np.empty((len(s), d))
    bad = _I64()
    code = lib().or_gather_adapter(_ptr(w_a), _ptr(w_b), _I64(d), _I64(r), _ptr(s), _I64(len(s)), _ptr(wak),
                                   _ptr(wbk), C.byref(bad))
    if code:
        raise OracleError(code, str(bad.value))
    return wak, wbk


def matmul(a, b):
    a, b = _f64(a), _f64(b)
    out = np.empty((a.shape[0], b.shape[1]))
    lib().or_matmul(_ptr(a), _ptr(b), _I64(a.shape[0]), _I64(a.shape[1]), _I64(b.shape[1]), _ptr(out))
    return out


def _base(d, w_in, w_out):
    if w_in is None:
        return np.zeros((d, 0)), np.zeros((0, d)), 0
    return _f64(w_in), _f64(w_out), w_in.shape[1]


def ffn_forward(h, w_a_k, w_b_k, w_in=None, w_out=None, act=0):
    h, w_a_k, w_b_k = _f64(h), _f64(w_a_k), _f64(w_b_k)
    T, d = h.shape
    w_in, w_out, n = _base(d, w_in, w_out)
    s = w_a_k.shape[1]
    out = np.empty((T, d))
    z = np.empty((T, s))
    pre = np.empty((T, n))
    lib().or_ffn_forward(_ptr(h), _I64(T), _I64(d), _ptr(w_in), _ptr(w_out), _I64(n), C.c_int(act), _ptr(w_a_k),
                         _ptr(w_b_k), _I64(s), _ptr(out), _ptr(z), _ptr(pre))
    return out, z, pre


def router_ste(h, z, w_b_k, s, tau, grad_out, esz, n_experts):
    """trainer.cpp:140-181 stage_router_ste -> (grad_g [N x d], touched [N] bool)."""
    h, z, w_b_k, grad_out = map(_f64, (h, z, w_b_k, grad_out))
    s, tau = _i64(s), _i64(tau)
    T, d = h.shape
    gg = np.zeros((n_experts, d))
    touched = np.zeros(n_experts, np.int8)
    lib().or_router_ste(_ptr(h), _ptr(z), _ptr(w_b_k), _ptr(s), _I64(len(s)), _ptr(tau), _I64(tau.shape[1]),
                        _ptr(grad_out), _I64(T), _I64(d), _I64(esz), _ptr(gg), _ptr(touched))
    return gg, touched.astype(bool)


def ffn_backward(grad_out, h, z, base_pre, w_a_k, w_b_k, w_in=None, w_out=None, act=0):
    grad_out, h, z, w_a_k, w_b_k = map(_f64, (grad_out, h, z, w_a_k, w_b_k))
    T, d = h.shape
    w_in, w_out, n = _base(d, w_in, w_out)
    base_pre = _f64(base_pre) if base_pre is not None else np.zeros((T, n))
    s = w_a_k.shape[1]
    gwa = np.empty((d, s))
    gwb = np.empty((s, d))
    gh = np.empty((T, d))
    lib().or_ffn_backward(_ptr(grad_out), _ptr(h), _ptr(z), _ptr(base_pre), _I64(T), _I64(d), _ptr(w_in),
                          _ptr(w_out), _I64(n), C.c_int(act), _ptr(w_a_k), _ptr(w_b_k), _I64(s), _ptr(gwa),
                          _ptr(gwb), _ptr(gh))
    return gwa, gwb, gh


class OracleStore:
    """Arrays of one reference HostLayer (memtier.hpp:90-106) for the scatter/Adam restatement."""

    def __init__(self, w_a, w_b):
        self.w_a = _f64(w_a).copy()
        self.w_b = _f64(w_b).copy()
        d, r = self.w_a.shape
        self.d, self.r = d, r
        self.m_a = np.zeros((d, r))
        self.v_a = np.zeros((d, r))
        self.m_b = np.zeros((r, d))
        self.v_b = np.zeros((r, d))
        self.stage_a = np.zeros((d, r))
        self.stage_b = np.zeros((r, d))
        self.staged = np.zeros(r, np.int8)
        self.pair_step = np.zeros(r, np.int64)

    def scatter_grads(self, s, gwa, gwb):
        s, gwa, gwb = _i64(s), _f64(gwa), _f64(gwb)
        bad = _I64()
        code = lib().or_scatter_grads(_I64(self.d), _I64(self.r), _ptr(self.stage_a), _ptr(self.stage_b),
                                      _ptr(self.staged), _ptr(s), _I64(len(s)), _ptr(gwa), _ptr(gwb), C.byref(bad))
        if code:
            raise OracleError(code, str(bad.value))

    def sparse_adam(self, lr, beta1=0.9, beta2=0.999, eps=1e-8):
        lib().or_sparse_adam(_I64(self.d), _I64(self.r), _ptr(self.w_a), _ptr(self.w_b), _ptr(self.m_a),
                             _ptr(self.v_a), _ptr(self.m_b), _ptr(self.v_b), _ptr(self.stage_a), _ptr(self.stage_b),
                             _ptr(self.staged), _ptr(self.pair_step), _D(beta1), _D(beta2), _D(eps), _D(lr))


# ------------------------------------------------------------ reference (ref_*)

def ref_ke_select(h, w_g, w_a, kk, k):
    h, w_g, w_a = _f64(h), _f64(w_g), _f64(w_a)
    T, d = h.shape
    N = w_g.shape[0]
    r = w_a.shape[1]
    kk_eff = min(kk, N)
    cap = max(1, min(k, kk_eff * (r // max(N, 1))))
    per = np.empty((T, cap), np.int64)
    tau = np.empty((T, kk_eff), np.int64)
    uni = np.empty(r, np.int64)
    us, take = _I64(), _I64()
    _check_ref(ref().ref_ke_select(_ptr(h), _I64(T), _I64(d), _ptr(w_g), _I64(N), _ptr(w_a), _I64(r), _I64(kk),
                                   _I64(k), _ptr(per), _ptr(tau), _ptr(uni), C.byref(us), C.byref(take)))
    return dict(per_token=per[:, : take.value].copy(), tau=tau, unioned=uni[: us.value].copy(), take=take.value)


def ref_topk_select(h, w_a, k):
    h, w_a = _f64(h), _f64(w_a)
    T, d = h.shape
    r = w_a.shape[1]
    per = np.empty((T, max(1, min(k, r))), np.int64)
    uni = np.empty(r, np.int64)
    us, take = _I64(), _I64()
    _check_ref(ref().ref_topk_select(_ptr(h), _I64(T), _I64(d), _ptr(w_a), _I64(r), _I64(k), _ptr(per), _ptr(uni),
                                     C.byref(us), C.byref(take)))
    return dict(per_token=per[:, : take.value].copy(), unioned=uni[: us.value].copy(), take=take.value)


def ref_ffn_forward(h, w_a_k, w_b_k, w_in=None, w_out=None, act=0):
    h, w_a_k, w_b_k = _f64(h), _f64(w_a_k), _f64(w_b_k)
    T, d = h.shape
    w_in, w_out, n = _base(d, w_in, w_out)
    s = w_a_k.shape[1]
    out, z, pre = np.empty((T, d)), np.empty((T, s)), np.empty((T, n))
    _check_ref(ref().ref_ffn_forward(_ptr(h), _I64(T), _I64(d), _ptr(w_in), _ptr(w_out), _I64(n), C.c_int(act),
                                     _ptr(w_a_k), _ptr(w_b_k), _I64(s), _ptr(out), _ptr(z), _ptr(pre)))
    return out, z, pre


def ref_ffn_backward(h, w_a_k, w_b_k, grad_out, w_in=None, w_out=None, act=0):
    h, w_a_k, w_b_k, grad_out = map(_f64, (h, w_a_k, w_b_k, grad_out))
    T, d = h.shape
    w_in, w_out, n = _base(d, w_in, w_out)
    s = w_a_k.shape[1]
    gwa, gwb, gh = np.empty((d, s)), np.empty((s, d)), np.empty((T, d))
    _check_ref(ref().ref_ffn_backward(_ptr(h), _I64(T), _I64(d), _ptr(w_in), _ptr(w_out), _I64(n), C.c_int(act),
                                      _ptr(w_a_k), _ptr(w_b_k), _I64(s), _ptr(grad_out), _ptr(gwa), _ptr(gwb),
                                      _ptr(gh)))
    return gwa, gwb, gh


class RefStore:
    """The reference HostStore (memtier.hpp:108-133), driven through its public API."""

    TENSORS = {"w_a": 0, "w_b": 1, "w_g": 2, "m_a": 3, "v_a": 4, "m_b": 5, "v_b": 6, "stage_a": 7, "stage_b": 8}

    def __init__(self, layers, d, r, n_experts, seed=1, train_router=False):
        self.layers, self.d, self.r, self.n = layers, d, r, n_experts
        self.h = ref().ref_store_init(layers, d, r, n_experts, int(train_router), seed)
        if not self.h:
            raise OracleError(9, ref().ref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            ref().ref_store_free(self.h)
            self.h = None

    def _shape(self, name):
        return {"w_a": (self.d, self.r), "m_a": (self.d, self.r), "v_a": (self.d, self.r),
                "stage_a": (self.d, self.r), "w_g": (self.n, self.d)}.get(name, (self.r, self.d))

    def get(self, layer, name):
        out = np.empty(self._shape(name))
        _check_ref(ref().ref_store_get(_P(self.h), _I64(layer), C.c_int(self.TENSORS[name]), _ptr(out)))
        return out

    def set(self, layer, name, value):
        value = _f64(value)
        assert value.shape == self._shape(name)
        _check_ref(ref().ref_store_set(_P(self.h), _I64(layer), C.c_int(self.TENSORS[name]), _ptr(value)))

    def pair_step(self, layer):
        out = np.empty(self.r, np.int64)
        _check_ref(ref().ref_store_pair_step(_P(self.h), _I64(layer), _ptr(out)))
        return out

    def staged(self, layer):
        out = np.empty(self.r, np.int8)
        _check_ref(ref().ref_store_staged(_P(self.h), _I64(layer), _ptr(out)))
        return out

    def scatter_grads(self, layer, s, gwa, gwb):
        s, gwa, gwb = _i64(s), _f64(gwa), _f64(gwb)
        m = _I64()
        _check_ref(ref().ref_scatter_grads(_P(self.h), _I64(layer), _ptr(s), _I64(len(s)), _ptr(gwa), _ptr(gwb),
                                           C.byref(m)))
        return m.value

    def save(self, path, extra="{}", step=0):
        """The reference's save_checkpoint (MEFT1) of this store."""
        _check_ref(ref().ref_store_save(_P(self.h), str(path).encode(), extra.encode(), _I64(step)))

    def stage_router_grads(self, layer, rows, grad_rows):
        rows, grad_rows = _i64(rows), _f64(grad_rows)
        _check_ref(ref().ref_stage_router_grads(_P(self.h), _I64(layer), _ptr(rows), _I64(len(rows)),
                                                _ptr(grad_rows)))

    def router(self, layer):
        """(w_g, m_g, v_g, router_step) of the layer."""
        w, m, v = (np.empty((self.n, self.d)) for _ in range(3))
        st = np.empty(self.n, np.int64)
        _check_ref(ref().ref_store_router(_P(self.h), _I64(layer), _ptr(w), _ptr(m), _ptr(v), _ptr(st)))
        return w, m, v, st

    def sparse_adam(self, layer, lr, beta1=0.9, beta2=0.999, eps=1e-8):
        _check_ref(ref().ref_sparse_adam(_P(self.h), _I64(layer), _D(beta1), _D(beta2), _D(eps), _D(lr)))

    def step_phases(self, layer, h, grad_out, kk, k, lr, row_slices):
        """The layer step of the T-token batch (h, grad_out) through the reference's public API in its phases:
        push_hidden + ke_select + fetch on the whole batch, sparse_ffn_pa + sparse_backward on each (lo, hi) row
        slice of the batch against that union, then scatter_grads + sparse_adam_update of the union (ref_capi.cpp
        ref_step_*). Returns the phase seconds (per-slice lists for forward / backward) and |S|."""
        h, grad_out = _f64(h), _f64(grad_out)
        T = h.shape[0]
        sel_s, fetch_s, us = _D(), _D(), _I64()
        st = ref().ref_step_begin(_P(self.h), _I64(layer), _ptr(h), _I64(T), _I64(kk), _I64(k), C.byref(sel_s),
                                  C.byref(fetch_s), C.byref(us))
        if not st:
            raise OracleError(9, ref().ref_last_error().decode())
        fwd, bwd = [], []
        try:
            for lo, hi in row_slices:
                f, b = _D(), _D()
                _check_ref(ref().ref_step_rows(_P(st), _ptr(h[lo:hi]), _ptr(grad_out[lo:hi]), _I64(hi - lo),
                                               C.byref(f), C.byref(b)))
                fwd.append(f.value)
                bwd.append(b.value)
        finally:
            sc, ad = _D(), _D()
            _check_ref(ref().ref_step_finish(_P(st), _P(self.h), _D(lr), C.byref(sc), C.byref(ad)))
        return dict(select=sel_s.value, fetch=fetch_s.value, forward=fwd, backward=bwd, scatter=sc.value,
                    adam=ad.value, union_size=us.value)

    def layer_step(self, layer, h, grad_out, kk, k, lr, want_outputs=True):
        h, grad_out = _f64(h), _f64(grad_out)
        T = h.shape[0]
        out = np.empty((T, self.d)) if want_outputs else None
        gh = np.empty((T, self.d)) if want_outputs else None
        us = _I64()
        phases = np.zeros(6)
        _check_ref(ref().ref_layer_step(_P(self.h), _I64(layer), _ptr(h), _I64(T), _ptr(grad_out), _I64(kk), _I64(k),
                                        _D(lr), _ptr(out), _ptr(gh), C.byref(us), _ptr(phases)))
        return dict(out=out, grad_h=gh, union_size=us.value, phases=phases)
