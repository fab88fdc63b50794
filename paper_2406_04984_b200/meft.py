"""Python mirror of the reference MEFT hot-path API over the C ABI (include/meft_cuda.h).

Names and argument meaning follow the reference (proj/include/meft/*.hpp): ``ke_select``, ``topk_select``,
``route_scores``, ``select_experts``, ``gather_adapter``, ``sparse_ffn_pa`` (adapter half: ``ffn_forward``),
``sparse_backward`` (``ffn_backward``), ``fetch``, ``scatter_grads``, ``sparse_adam_update``; errors raise
``MeftError`` whose ``kind`` is the reference exception type. torch is used only for device memory and the
stream; every computation is a kernel of libmeft_cuda.so. Key tables are neuron-major ([pairs x d]).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import BF16, F32, F64, STORE_COMPACT, STORE_F64, STORE_MIXED, TENSORS, CkptHeader, MeftError, check, lib

P = C.c_void_p
I64 = C.c_int64

_DT = {torch.float64: F64, torch.float32: F32, torch.bfloat16: BF16}


def _p(t):
    return None if t is None else P(t.data_ptr())


def _dt(t):
    try:
        return _DT[t.dtype]
    except KeyError:
        raise MeftError(2, f"unsupported dtype {t.dtype}") from None


def _contig(*ts):
    for t in ts:
        if t is not None and (not t.is_cuda or not t.is_contiguous()):
            raise MeftError(2, "tensors must be contiguous CUDA tensors")


class _CAI:
    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


class Context:
    """meft_ctx bound to torch's current stream of `device` (so torch.cuda.Event timing sees our kernels)."""

    def __init__(self, device: int = 0, stream: torch.cuda.Stream | None = None):
        torch.cuda.set_device(device)
        self.device = device
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        h = P()
        check(lib().meft_ctx_create(device, P(self.stream.cuda_stream), C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().meft_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, status):
        check(status, self.h)

    def synchronize(self):
        self.check(lib().meft_synchronize(self.h))

    PHASES = ("select", "gather", "ffn_forward", "ffn_backward", "adam")

    def set_selection(self, exact: bool):
        """exact=True forces fp64 SIMT scoring of every candidate (cross-validation of the certified path)."""
        self.check(lib().meft_ctx_set_selection(self.h, 1 if exact else 0))

    def set_gather(self, mode: str):
        """How the fused step's GEMMs read the selected key/value rows: "auto", "kernel" or "tma"."""
        self.check(lib().meft_ctx_set_gather(self.h, {"auto": 0, "kernel": 1, "tma": 2}[mode]))

    def set_adam(self, mode: str):
        """Fused layer step's sparse Adam: "epilogue" (in the weight-gradient GEMMs) or "pass" (separate kernel)."""
        self.check(lib().meft_ctx_set_adam(self.h, {"epilogue": 0, "pass": 1}[mode]))

    def set_check_finite(self, on: bool):
        """Fused layer steps raise the reference's 'non-finite' error on NaN / Inf in out or grad_h."""
        self.check(lib().meft_ctx_set_check_finite(self.h, int(on)))

    def set_host_sync(self, on):
        """on=False: fused layer steps never wait for the device (the FFN GEMMs read |S| on the device), so steps
        enqueue back to back and can be captured (graph()); on=True reads |S| back mid-step and sizes the GEMMs on
        the host; on=None (the default, MEFT_HOST_SYNC_AUTO): the first for dense unions, the second otherwise.
        Bit-identical results (meft_ctx_set_host_sync)."""
        self.check(lib().meft_ctx_set_host_sync(self.h, -1 if on is None else int(bool(on))))

    def graph(self):
        """Capture the enqueue-only calls made inside `with ctx.graph() as g:` into a CUDA graph; g.replay()
        re-runs them on the context stream. Run the same calls once eagerly first (scratch buffers must exist)."""
        return Graph(self)

    def set_timing(self, on: bool):
        self.check(lib().meft_ctx_set_timing(self.h, int(on)))

    def read_timing(self):
        """{phase: (ms, launches)} accumulated since the last read (CUDA events on the ctx stream)."""
        ms = (C.c_double * 5)()
        ln = (C.c_int64 * 5)()
        self.check(lib().meft_ctx_read_timing(self.h, ms, ln))
        return {p: (ms[i], ln[i]) for i, p in enumerate(self.PHASES)}


class Graph:
    """A CUDA graph of context-stream work (meft_graph_begin / end / launch)."""

    def __init__(self, ctx: Context):
        self.ctx = ctx
        self.h = None

    def __enter__(self):
        self.ctx.check(lib().meft_graph_begin(self.ctx.h))
        return self

    def __exit__(self, exc_type, exc, tb):
        h = P()
        st = lib().meft_graph_end(self.ctx.h, C.byref(h))
        if exc_type is None:
            self.ctx.check(st)
            self.h = h
        elif h:
            lib().meft_graph_destroy(h)
        return False

    def replay(self):
        self.ctx.check(lib().meft_graph_launch(self.ctx.h, self.h))

    def close(self):
        if getattr(self, "h", None):
            lib().meft_graph_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def kernel_launches() -> int:
    """Kernels libmeft_cuda.so has launched from this thread so far."""
    return int(lib().meft_kernel_launches())


def reference_uniform(seed: int, stream: int, shape, lo: float, hi: float, bf16: bool = False) -> np.ndarray:
    """SeededRng(mix_seed(seed, stream)).uniform_matrix(*shape, lo, hi) of the reference (rng.hpp:13-21, 62-66) as a
    float64 host array, optionally bf16-rounded: the BASELINE.md §3 input streams (W_B 0x7001, h 0x7002, grad_out
    0x7003) that bench.py's GPU and CPU arms share."""
    out = np.empty(tuple(shape), np.float64)
    check(lib().meft_reference_uniform(C.c_uint64(seed), C.c_uint64(stream), out.size, lo, hi, int(bf16),
                                       out.ctypes.data_as(P)))
    return out


def selection_shape(M, N, kk, k):
    take, kk_eff, warn = I64(), I64(), C.c_int()
    check(lib().meft_selection_shape(M, N, kk, k, C.byref(take), C.byref(kk_eff), C.byref(warn)))
    return take.value, kk_eff.value, bool(warn.value)


def route_scores(ctx: Context, h, w_g):
    _contig(h, w_g)
    T, d = h.shape
    N = w_g.shape[0]
    out = torch.empty((T, N), dtype=torch.float64, device=h.device)
    ctx.check(lib().meft_route_scores(ctx.h, _dt(h), _p(h), _p(w_g), T, d, N, _p(out)))
    return out


def select_experts(ctx: Context, scores, kk):
    _contig(scores)
    T, N = scores.shape
    tau = torch.empty((T, max(1, min(kk, N))), dtype=torch.int32, device=scores.device)
    ctx.check(lib().meft_select_experts(ctx.h, _p(scores), T, N, kk, _p(tau)))
    return tau


@dataclass
class Selection:
    per_token: torch.Tensor  # [T x take] int32, rows ascending
    unioned: torch.Tensor    # [|S|] int32 ascending
    tau: torch.Tensor | None
    take: int
    warned: bool
    budget: int


def ke_select(ctx: Context, h, w_g, keys, kk: int, k: int, with_tau: bool = True) -> Selection:
    """ke_select (experts.cpp:47-117); keys neuron-major [M x d]; h/w_g/keys all f64 or all bf16."""
    _contig(h, w_g, keys)
    T, d = h.shape
    N, M = w_g.shape[0], keys.shape[0]
    if w_g.shape[1] != d or keys.shape[1] != d:
        raise MeftError(1, "ke_select: model dim mismatch")
    take, kk_eff, warned = selection_shape(M, N, kk, k)
    dev = h.device
    per = torch.empty((T, take), dtype=torch.int32, device=dev)
    tau = torch.empty((T, kk_eff), dtype=torch.int32, device=dev) if with_tau else None
    uni = torch.empty(M, dtype=torch.int32, device=dev)
    usz = torch.zeros(1, dtype=torch.int32, device=dev)
    ctx.check(lib().meft_ke_select(ctx.h, _dt(h), _p(h), _p(w_g), _p(keys), T, d, M, N, kk, k, _p(per), _p(tau),
                                   _p(uni), _p(usz)))
    n = int(usz.item())
    return Selection(per, uni[:n], tau, take, warned, k)


def topk_select(ctx: Context, h, keys, k: int) -> Selection:
    """topk_select (adapter.cpp:42-84)."""
    _contig(h, keys)
    T, d = h.shape
    M = keys.shape[0]
    if k < 1:
        raise MeftError(2, "topk_select: K must be >= 1")
    take = min(k, M)
    dev = h.device
    per = torch.empty((T, take), dtype=torch.int32, device=dev)
    uni = torch.empty(M, dtype=torch.int32, device=dev)
    usz = torch.zeros(1, dtype=torch.int32, device=dev)
    ctx.check(lib().meft_topk_select(ctx.h, _dt(h), _p(h), _p(keys), T, d, M, k, _p(per), _p(uni), _p(usz)))
    n = int(usz.item())
    return Selection(per, uni[:n], None, take, k > M, k)


def gather_adapter(ctx: Context, keys, values, S):
    """gather_adapter (adapter.cpp:86-110) on neuron-major tables."""
    _contig(keys, values, S)
    M, d = keys.shape
    s = S.numel()
    ks = torch.empty((s, d), dtype=keys.dtype, device=keys.device)
    vs = torch.empty((s, d), dtype=values.dtype, device=values.device)
    ctx.check(lib().meft_gather_adapter(ctx.h, _dt(keys), _p(keys), _p(values), M, d, _p(S), s, _p(ks), _p(vs)))
    return ks, vs


def _ld(s):
    return max(8, (s + 63) // 64 * 64)


def ffn_forward(ctx: Context, h, keys_s, values_s, out=None, accumulate=False):
    """Adapter term of sparse_ffn_pa (adapter.cpp:122-126). Returns (z_or_act [T x ld], out, ld)."""
    _contig(h, keys_s, values_s)
    T, d = h.shape
    s = keys_s.shape[0]
    dt = _dt(h)
    ld = s if dt == F64 else _ld(s)
    z = torch.empty((T, max(ld, 1)), dtype=h.dtype, device=h.device)
    if out is None:
        out = torch.empty((T, d), dtype=torch.float64 if dt == F64 else torch.float32, device=h.device)
    ctx.check(lib().meft_ffn_forward(ctx.h, dt, _p(h), _p(keys_s), _p(values_s), T, d, s, ld, _p(z), _p(out),
                                     int(accumulate)))
    return z, out, ld


def ffn_backward(ctx: Context, grad_out, h, z, keys_s, values_s, ld, grad_h=None, accumulate_grad_h=False):
    """Adapter term of sparse_backward (adapter.cpp:166-175). Returns (grad_keys_s, grad_values_s, grad_h);
    grad_keys_s is neuron-major [s x d] (the transpose of the reference's d x s grad_w_a_k)."""
    _contig(grad_out, h, z, keys_s, values_s)
    T, d = h.shape
    s = keys_s.shape[0]
    dt = _dt(h)
    gdt = torch.float64 if dt == F64 else torch.float32
    masked = torch.empty_like(z)
    gk = torch.empty((s, d), dtype=gdt, device=h.device)
    gv = torch.empty((s, d), dtype=gdt, device=h.device)
    if grad_h is None:
        grad_h = torch.empty((T, d), dtype=gdt, device=h.device)
    ctx.check(lib().meft_ffn_backward(ctx.h, dt, _p(grad_out), _p(h), _p(z), _p(keys_s), _p(values_s), T, d, s, ld,
                                      _p(masked), _p(gk), _p(gv), _p(grad_h), int(accumulate_grad_h)))
    return gk, gv, grad_h


def matmul_f64(ctx: Context, a, b):
    _contig(a, b)
    out = torch.empty((a.shape[0], b.shape[1]), dtype=torch.float64, device=a.device)
    ctx.check(lib().meft_matmul_f64(ctx.h, _p(a), _p(b), a.shape[0], a.shape[1], b.shape[1], _p(out)))
    return out


class Store:
    """HBM-resident HostStore (memtier.hpp:108-133). precision: STORE_F64 (API fidelity), STORE_MIXED, or
    STORE_COMPACT (MIXED with bf16 Adam moments)."""

    def __init__(self, ctx: Context, layers, d, pairs, experts, precision=STORE_MIXED):
        self.ctx = ctx
        self.layers, self.d, self.pairs, self.experts, self.precision = layers, d, pairs, experts, precision
        h = P()
        ctx.check(lib().meft_store_create(ctx.h, layers, d, pairs, experts, precision, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().meft_store_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @classmethod
    def load(cls, ctx: Context, path, precision=STORE_MIXED):
        """load_checkpoint (MEFT1, memtier.cpp:328-396) straight into a new HBM store. Returns (store, header,
        extra_json)."""
        h, hdr, extra = P(), CkptHeader(), C.create_string_buffer(1 << 20)
        ctx.check(lib().meft_store_load(ctx.h, str(path).encode(), precision, C.byref(h), C.byref(hdr), extra,
                                        len(extra)))
        st = cls.__new__(cls)
        st.ctx, st.h = ctx, h
        st.layers, st.d, st.pairs, st.experts, st.precision = hdr.layers, hdr.dim, hdr.pairs, hdr.experts, precision
        return st, hdr, extra.value.decode()

    def save(self, path, step: int = 0, extra: str = "{}"):
        """save_checkpoint (MEFT1, memtier.cpp:288-326) of this HBM store."""
        self.ctx.check(lib().meft_store_save(self.ctx.h, self.h, str(path).encode(), step, extra.encode()))

    def expert_histogram(self, layer, reset=False):
        """Routed-token counts per expert accumulated by the fused steps (trainer.cpp:240)."""
        out = np.empty(self.experts, np.int64)
        self.ctx.check(lib().meft_store_expert_histogram(self.ctx.h, self.h, layer, out.ctypes.data_as(P),
                                                         int(reset)))
        return out

    def enable_router(self):
        """train_router state (m_g, v_g, router_step) for every layer."""
        self.ctx.check(lib().meft_store_enable_router(self.ctx.h, self.h))

    def init_reference(self, seed: int = 1):
        self.ctx.check(lib().meft_store_init_reference(self.ctx.h, self.h, C.c_uint64(seed)))

    def _ref_shape(self, name):
        if name in ("w_a", "m_a", "v_a", "stage_a"):
            return (self.d, self.pairs)
        if name == "w_g":
            return (self.experts, self.d)
        if name in ("m_g", "v_g"):
            return (self.experts, self.d)
        if name == "router_step":
            return (self.experts,)
        if name in ("pair_step", "staged"):
            return (self.pairs,)
        return (self.pairs, self.d)

    def upload(self, layer, name, host):
        dtype = {"pair_step": np.int64, "router_step": np.int64, "staged": np.int8}.get(name, np.float64)
        a = np.ascontiguousarray(host, dtype=dtype)
        shape = self._ref_shape(name)
        if a.shape != shape:
            raise MeftError(1, f"upload {name}: expected {shape}, got {a.shape}")
        rows, cols = (shape[0], 1) if len(shape) == 1 else shape
        self.ctx.check(lib().meft_store_upload_host(self.ctx.h, self.h, layer, TENSORS[name], a.ctypes.data_as(P),
                                                    rows, cols))

    def download(self, layer, name):
        dtype = {"pair_step": np.int64, "router_step": np.int64, "staged": np.int8}.get(name, np.float64)
        shape = self._ref_shape(name)
        a = np.empty(shape, dtype=dtype)
        rows, cols = (shape[0], 1) if len(shape) == 1 else shape
        self.ctx.check(lib().meft_store_download_host(self.ctx.h, self.h, layer, TENSORS[name], a.ctypes.data_as(P),
                                                      rows, cols))
        return a

    def tensor(self, layer, name) -> torch.Tensor:
        """Zero-copy torch view of a store tensor in its DEVICE layout (neuron-major [pairs x d])."""
        ptr, dt, r, c = P(), C.c_int(), I64(), I64()
        check(lib().meft_store_tensor(self.h, layer, TENSORS[name], C.byref(ptr), C.byref(dt), C.byref(r),
                                      C.byref(c)))
        if name == "pair_step":
            return torch.as_tensor(_CAI(ptr.value, (r.value,), "<i4"), device=f"cuda:{self.ctx.device}")
        if name == "staged":
            return torch.as_tensor(_CAI(ptr.value, (r.value,), "|u1"), device=f"cuda:{self.ctx.device}")
        ts = {F64: "<f8", F32: "<f4", BF16: "<u2"}[dt.value]
        t = torch.as_tensor(_CAI(ptr.value, (r.value, c.value), ts), device=f"cuda:{self.ctx.device}")
        return t.view(torch.bfloat16) if dt.value == BF16 else t

    def fetch(self, layer, S):
        _contig(S)
        s = S.numel()
        dt = torch.float64 if self.precision == STORE_F64 else torch.bfloat16
        ks = torch.empty((s, self.d), dtype=dt, device=S.device)
        vs = torch.empty((s, self.d), dtype=dt, device=S.device)
        self.ctx.check(lib().meft_fetch(self.ctx.h, self.h, layer, _p(S), s, _p(ks), _p(vs)))
        return ks, vs

    def scatter_grads(self, layer, S, grad_keys_s, grad_values_s):
        _contig(S, grad_keys_s, grad_values_s)
        self.ctx.check(lib().meft_scatter_grads(self.ctx.h, self.h, layer, _p(S), S.numel(), _p(grad_keys_s),
                                                _p(grad_values_s), _dt(grad_keys_s)))

    def sparse_adam_update(self, layer, lr, beta1=0.9, beta2=0.999, eps=1e-8):
        self.ctx.check(lib().meft_sparse_adam_update(self.ctx.h, self.h, layer, beta1, beta2, eps, lr))

    def layer_step(self, layer, h, grad_out, kk, k, lr, beta1=0.9, beta2=0.999, eps=1e-8, out=None, grad_h=None,
                   want_selection=False, base=None, want_info=True, per_token=None, union=None):
        """meft_ffn -> sparse_backward -> scatter_grads -> sparse_adam_update on device buffers (bf16 in).
        base = (w_in bf16 [d x n], w_out bf16 [n x d], act 0 SiLU / 1 ReLU): the frozen base FFN as well.
        want_info=False passes no meft_step_info (with host sync off the step then never synchronises; returns
        None); per_token / union: caller-owned int32 outputs ([T x take], [M]) instead of fresh ones."""
        _contig(h, grad_out)
        T, d = h.shape
        take, _, _ = selection_shape(self.pairs, self.experts, kk, k)
        per = per_token if per_token is not None else (
            torch.empty((T, take), dtype=torch.int32, device=h.device) if want_selection else None)
        uni = union if union is not None else (
            torch.empty(self.pairs, dtype=torch.int32, device=h.device) if want_selection else None)
        info = _lib.StepInfo()
        info_p = C.byref(info) if want_info else None
        if base is None:
            self.ctx.check(lib().meft_layer_step(self.ctx.h, self.h, layer, _p(h), _p(grad_out), T, kk, k, beta1,
                                                 beta2, eps, lr, _p(out), _p(grad_h), _p(per), _p(uni), info_p))
        else:
            w_in, w_out, act = base
            _contig(w_in, w_out)
            bf = _lib.BaseFfn(w_in.data_ptr(), w_out.data_ptr(), w_in.shape[1], act)
            self.ctx.check(lib().meft_layer_step_base(self.ctx.h, self.h, layer, _p(h), _p(grad_out), T, kk, k, beta1,
                                                      beta2, eps, lr, _p(out), _p(grad_h), _p(per), _p(uni),
                                                      info_p, C.byref(bf)))
        if not want_info:
            return None
        res = {name: getattr(info, name) for name, _ in _lib.StepInfo._fields_}
        res["warned"] = bool(info.warned)
        if want_selection:
            res["per_token"] = per
            res["unioned"] = uni[: info.union_size]
        return res

    def layer_step_host(self, layer, h_host, g_host, kk, k, lr, out_host=None, grad_h_host=None, beta1=0.9,
                        beta2=0.999, eps=1e-8):
        """Same step from host (CPU, ideally pinned) bf16 tensors; results land in host f32 tensors."""
        T = h_host.shape[0]
        info = _lib.StepInfo()
        self.ctx.check(lib().meft_layer_step_host(self.ctx.h, self.h, layer, _p(h_host), _p(g_host), T, kk, k, beta1,
                                                  beta2, eps, lr, _p(out_host), _p(grad_h_host), C.byref(info)))
        return dict(union_size=info.union_size, take=info.take, gpu_launches=info.gpu_launches)
