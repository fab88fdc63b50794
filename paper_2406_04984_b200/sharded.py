"""Expert-sharded MEFT layer step over P ranks (one per GPU), DESIGN.md §6.

Rank r owns experts [r*N/P, (r+1)*N/P) and their M/P key/value pairs (+ Adam state); the router W_g is
replicated. Each rank brings its own T tokens (weak scaling: the layer step is over all P*T tokens, with the
reference's batch-union semantics). Per step:

  1. route the local tokens (certified, exact tau) ............................ home rank
  2. all-to-all: dispatch (token id, expert) entries to the expert's owner, who gathers the token rows from the
     all-gathered h (step 8a, started first) ..................................... NCCL
  3. approximate candidate scores against the owner's keys (tcgen05) ............ owner rank
  4. all-to-all: candidate scores back; all-gather key norms .................... NCCL
  5. certified top-K classification (sure / ambiguous) .......................... home rank
  6. all-to-all: ambiguous (row, key) requests -> owners' exact fp64 scores -> back  NCCL + owner
  7. finalize the per-token selection; all-reduce(MAX) of the M-byte union bitmap .. home + NCCL
  8. all-gather h and grad_out; FFN + fused scatter + lazy Adam on the local part of the union .. owner
  9. reduce-scatter the partial out / grad_h back to the token homes ............. NCCL

Selection is the single-GPU certified algorithm split at the rank boundary, so indices are the reference's,
bit for bit. The compute is behind an engine interface: ``DeviceEngine`` calls libmeft_cuda.so; the CPU test
suite drives the same orchestration with an fp64 oracle engine over gloo (tests/test_sharded.py).
torch is used for buffers, index bookkeeping (argsort/bincount of routing decisions) and torch.distributed.
"""
from __future__ import annotations

import ctypes as C
import math
import os

import torch
import torch.distributed as dist

from . import _lib
from ._lib import check, lib


def cert_bound_coeff(d: int) -> float:
    """CB(d) of select_tc.cuh: |approx - reference| <= CB(d) * ||h|| * ||w||."""
    return 32.0 * 2.0 ** -24 * ((d + 15) // 16 + 1) + d * 2.0 ** -52


def _p(t):
    return None if t is None else C.c_void_p(t.data_ptr())


class TorchGlue:
    """The protocol's index bookkeeping as framework ops -- the reference semantics of the device plan kernels
    (csrc/shard_plan.cu), used by engines without them (the CPU test engine). All orders are stable."""

    def dispatch(self, tau, h, n_loc, P, rows=True):
        """(token, slot) rows bucketed by expert owner: send rows / owner-local experts in bucket order, order[p] =
        flat (t*kk + s) index, inv = its inverse, rows per owner."""
        kk = tau.shape[1]
        flat = tau.reshape(-1).long()
        owner = flat // n_loc
        order = torch.argsort(owner, stable=True)
        inv = torch.empty_like(order)
        inv[order] = torch.arange(order.numel(), device=order.device)
        counts = torch.bincount(owner, minlength=P).tolist()
        send_exp = (flat[order] - owner[order] * n_loc).to(torch.int32)
        return h[order // kk], send_exp, order.to(torch.int32), inv.to(torch.int32), counts

    def unpermute(self, src, order):
        out = torch.empty_like(src)
        out[order.long()] = src
        return out

    def gather_rows(self, src, idx):
        return src[idx.long()]

    def requests(self, amb, n_amb, tau, inv, E, M_loc, P, row_base):
        """Exact re-scoring requests of the ambiguous candidates, bucketed by key owner in (token, position) order:
        (owner receive row, owner-local key, back index t*C + a, requests per owner, total)."""
        T, C = amb.shape
        kk = tau.shape[1]
        dev = amb.device
        na = n_amb.long()
        n = int(na.sum().item())
        tok = torch.repeat_interleave(torch.arange(T, device=dev), na)
        pos = torch.arange(n, device=dev) - torch.repeat_interleave(torch.cumsum(na, 0) - na, na)
        gidx = amb[tok, pos].long()
        slot = (tau[tok].long() == (gidx // E)[:, None]).int().argmax(1)
        owner = gidx // M_loc
        row = inv[tok * kk + slot].long() + torch.tensor(row_base, device=dev)[owner]
        key = gidx - owner * M_loc
        order = torch.argsort(owner, stable=True)
        counts = torch.bincount(owner, minlength=P).tolist()
        return (row[order].to(torch.int32), key[order].to(torch.int32), (tok * C + pos)[order].to(torch.int32),
                counts, n)

    def scatter_exact(self, x, back, T, C):
        xs = torch.zeros(T * C, dtype=torch.float64, device=x.device)
        xs[back.long()] = x
        return xs.view(T, C)


class DeviceEngine:
    """Per-rank compute on one B200 through the C ABI (the store holds this rank's expert shard)."""

    def __init__(self, ctx, store, w_g):
        self.ctx, self.store, self.w_g = ctx, store, w_g  # w_g: full replicated router, bf16 [N x d] on device
        self.dev = w_g.device

    def _check(self, st):
        self.ctx.check(st)

    # ---- protocol bookkeeping on the device (csrc/shard_plan.cu; semantics: TorchGlue)
    def dispatch(self, tau, h, n_loc, P, rows=True):
        T, kk = tau.shape
        d = h.shape[1]
        n = T * kk
        send_rows = torch.empty((n, d), dtype=h.dtype, device=self.dev) if rows else None
        send_exp = torch.empty(n, dtype=torch.int32, device=self.dev)
        order = torch.empty(n, dtype=torch.int32, device=self.dev)
        inv = torch.empty(n, dtype=torch.int32, device=self.dev)
        counts = (C.c_int64 * P)()
        self._check(lib().meft_shard_dispatch(self.ctx.h, _p(tau), T, kk, n_loc, P, _p(h), d, _p(send_rows),
                                              _p(send_exp), _p(order), _p(inv), counts))
        return send_rows, send_exp, order, inv, list(counts)

    def gather_rows(self, src, idx):
        """src[idx] (rows of a contiguous device tensor) by meft_gather_rows."""
        n = idx.numel()
        out = torch.empty((n,) + tuple(src.shape[1:]), dtype=src.dtype, device=self.dev)
        if n:
            row_bytes = src[0].numel() * src.element_size()
            self._check(lib().meft_gather_rows(self.ctx.h, _p(src), row_bytes, _p(idx), n, _p(out)))
        return out

    def unpermute(self, src, order):
        out = torch.empty_like(src)
        n = src.shape[0]
        self._check(lib().meft_shard_unpermute_rows(self.ctx.h, _p(src), _p(order), n, src.numel() // max(n, 1),
                                                    _p(out)))
        return out

    def requests(self, amb, n_amb, tau, inv, E, M_loc, P, row_base):
        T, Cc = amb.shape
        kk = tau.shape[1]
        cap = max(1, T * Cc)
        row = torch.empty(cap, dtype=torch.int32, device=self.dev)
        key = torch.empty(cap, dtype=torch.int32, device=self.dev)
        back = torch.empty(cap, dtype=torch.int32, device=self.dev)
        counts = (C.c_int64 * P)()
        total = C.c_int64()
        base = (C.c_int64 * P)(*row_base)
        self._check(lib().meft_shard_requests(self.ctx.h, _p(amb), _p(n_amb), _p(tau), _p(inv), T, Cc, kk, E, M_loc,
                                              P, base, _p(row), _p(key), _p(back), counts, C.byref(total)))
        n = total.value
        return row[:n], key[:n], back[:n], list(counts), n

    def scatter_exact(self, x, back, T, Cc):
        xs = torch.zeros((T, Cc), dtype=torch.float64, device=self.dev)
        if back.numel():
            self._check(lib().meft_shard_scatter_f64(self.ctx.h, _p(x), _p(back), back.numel(), _p(xs)))
        return xs

    def route(self, h, kk):
        T, d = h.shape
        N = self.w_g.shape[0]
        tau = torch.empty((T, min(kk, N)), dtype=torch.int32, device=self.dev)
        self._check(lib().meft_route_select(self.ctx.h, _p(h), _p(self.w_g), T, d, N, kk, _p(tau)))
        return tau

    def row_stats(self, rows):
        n, d = rows.shape
        norms = torch.empty(n, dtype=torch.float32, device=self.dev)
        lsb = torch.empty(n, dtype=torch.int32, device=self.dev)
        self._check(lib().meft_row_stats(self.ctx.h, _p(rows), n, d, _p(norms), _p(lsb)))
        return norms, lsb

    def key_stats(self):
        n = self.store.pairs
        norms = torch.empty(n, dtype=torch.float32, device=self.dev)
        lsb = torch.empty(n, dtype=torch.int32, device=self.dev)
        self._check(lib().meft_store_key_stats(self.ctx.h, self.store.h, 0, _p(norms), _p(lsb)))
        return norms, lsb

    def score(self, rows, expert_local):
        R = rows.shape[0]
        E = self.store.pairs // self.store.experts
        cand = torch.empty((R, E), dtype=torch.float32, device=self.dev)
        if R:
            self._check(lib().meft_score_candidates(self.ctx.h, self.store.h, 0, _p(rows), _p(expert_local), R,
                                                    _p(cand)))
        return cand

    def exact(self, rows, pair_row, pair_key):
        Q = pair_row.numel()
        out = torch.empty(Q, dtype=torch.float64, device=self.dev)
        if Q:
            self._check(lib().meft_exact_scores(self.ctx.h, self.store.h, 0, _p(rows), rows.shape[0], _p(pair_row),
                                                _p(pair_key), Q, _p(out)))
        return out

    def classify(self, cand, tau, hn, kn, take, d):
        T, Cc = cand.shape
        kk = tau.shape[1]
        E = Cc // kk
        sure = torch.empty((T, take), dtype=torch.int32, device=self.dev)
        n_sure = torch.empty(T, dtype=torch.int32, device=self.dev)
        amb = torch.empty((T, Cc), dtype=torch.int32, device=self.dev)
        n_amb = torch.empty(T, dtype=torch.int32, device=self.dev)
        self._check(lib().meft_topk_classify(self.ctx.h, _p(cand), _p(tau), T, kk, E, take, d, _p(hn), _p(kn),
                                             _p(sure), _p(n_sure), _p(amb), _p(n_amb)))
        return sure, n_sure, amb, n_amb

    def finalize(self, sure, n_sure, amb, n_amb, x, take, M):
        T, Cc = amb.shape
        per = torch.empty((T, take), dtype=torch.int32, device=self.dev)
        flags = torch.zeros(M, dtype=torch.uint8, device=self.dev)
        self._check(lib().meft_topk_finalize(self.ctx.h, _p(sure), _p(n_sure), _p(amb), _p(n_amb), _p(x), T, Cc, take,
                                             _p(per), _p(flags)))
        return per, flags

    def ffn_local(self, h_all, g_all, S_local, lr, betas=(0.9, 0.999), eps=1e-8, g_ready=None, fwd_done=None,
                  gh_done=None, peer=None):
        """Events (torch.cuda.Event, optional): the backward waits for g_ready; fwd_done / gh_done are recorded
        when out / grad_h are final, for reduce-scatters overlapped with the rest of the step. With `peer`
        (PeerExchange) the out / grad_h rows are pushed into the token homes' receive buffers instead and
        (None, None) is returned."""
        T, d = h_all.shape
        ev = [C.c_void_p(e.cuda_event) if e is not None else None for e in (g_ready, fwd_done, gh_done)]
        if peer is not None:
            self._check(lib().meft_layer_ffn_local(self.ctx.h, self.store.h, 0, _p(h_all), _p(g_all), T,
                                                   _p(S_local), S_local.numel(), betas[0], betas[1], eps, lr, None,
                                                   None, *ev, C.byref(peer.desc)))
            return None, None
        out = torch.empty((T, d), dtype=torch.float32, device=self.dev)
        gh = torch.empty((T, d), dtype=torch.float32, device=self.dev)
        self._check(lib().meft_layer_ffn_local(self.ctx.h, self.store.h, 0, _p(h_all), _p(g_all), T, _p(S_local),
                                               S_local.numel(), betas[0], betas[1], eps, lr, _p(out), _p(gh), *ev,
                                               None))
        return out, gh


class PeerExchange:
    """Receive buffers of the fused peer-memory reduce-scatter (meft_peer_out): out and grad_h, each
    [world x rows x d] fp32 per home rank, allocated with cudaMalloc and mapped into every rank of `group` through
    CUDA IPC (handles all-gathered over the group). ``desc`` is the meft_peer_out for this rank; ``reduce`` folds
    this home's slots in slot order. ``peers`` lets a single process stand in for several ranks (tests)."""

    def __init__(self, ctx, rows, d, group=None, world=None, rank=None, local=None, fail_local=False):
        self.ctx, self.rows, self.d = ctx, rows, d
        self.world = world if world is not None else dist.get_world_size(group)
        self.rank = rank if rank is not None else dist.get_rank(group)
        self.dev = torch.device("cuda", torch.cuda.current_device())
        nbytes = self.world * rows * d * 4
        self._own, self._opened = [], []
        if local is not None:  # single-process emulation: `local` = [(out_ptr, gh_ptr)] of every emulated rank
            bases = local
        else:
            # Local setup may fail on one rank only (allocation, IPC export). Every rank still joins the one
            # all_gather_object below -- a failed rank contributes None -- so the group's collectives stay matched
            # and every rank raises together instead of some waiting forever in the gather.
            mine, handles = [], None
            try:
                if fail_local:
                    raise RuntimeError("caller's local setup failed")
                for _ in range(2):
                    p = C.c_void_p()
                    check(lib().meft_device_alloc(ctx.h, nbytes, C.byref(p)), ctx.h)
                    self._own.append(p.value)
                    mine.append(p.value)
                handles = []
                for p in mine:
                    hb = (C.c_char * 64)()
                    check(lib().meft_ipc_handle(ctx.h, C.c_void_p(p), hb), ctx.h)
                    handles.append(bytes(hb))
            except Exception:
                handles = None
            every = [None] * self.world
            dist.all_gather_object(every, handles, group=group)
            if any(e is None for e in every):
                self.close()
                raise RuntimeError("peer exchange: a rank could not allocate or export its receive buffers")
            bases = []
            try:  # a failure here is agreed on by the caller (ShardedLayer._peer_exchange: all-reduce of a flag)
                for r, hs in enumerate(every):
                    if r == self.rank:
                        bases.append(tuple(mine))
                        continue
                    ptrs = []
                    for hbytes in hs:
                        p = C.c_void_p()
                        check(lib().meft_ipc_open(ctx.h, (C.c_char * 64).from_buffer_copy(hbytes), C.byref(p)),
                              ctx.h)
                        self._opened.append(p.value)
                        ptrs.append(p.value)
                    bases.append(tuple(ptrs))
            except Exception:
                self.close()
                raise
        self.desc = _lib.PeerOut()
        self.desc.world, self.desc.rank, self.desc.rows = self.world, self.rank, rows
        for r, (po, pg) in enumerate(bases):
            self.desc.out_recv[r] = po
            self.desc.grad_h_recv[r] = pg
        self.recv = bases[self.rank]  # this home's (out, grad_h) receive buffers

    def reduce(self, ctx, which):
        """Sum this home's slots (which: 0 = out, 1 = grad_h) into a new [rows x d] fp32 tensor on ctx's stream."""
        out = torch.empty((self.rows, self.d), dtype=torch.float32, device=self.dev)
        check(lib().meft_peer_reduce(ctx.h, C.c_void_p(self.recv[which]), self.world, self.rows, self.d, _p(out)),
              ctx.h)
        return out

    def close(self):
        for p in self._opened:
            lib().meft_ipc_close(self.ctx.h, C.c_void_p(p))
        for p in self._own:
            lib().meft_device_free(self.ctx.h, C.c_void_p(p))
        self._opened, self._own = [], []


class ThreadGroup:
    """In-process stand-in for a process group: P threads of ONE process, one per emulated rank, exchange
    finished device tensors at host-side rendezvous (a barrier), so no kernel ever waits on another rank's
    kernel -- the way to run the multi-rank device path with fewer GPUs than ranks. Each thread calls
    ``bind(rank)`` first; the layer's collectives then route here instead of torch.distributed."""

    def __init__(self, world):
        import threading
        self.world = world
        self._barrier = threading.Barrier(world)
        self._slots = [None] * world
        self._local = threading.local()

    def bind(self, rank):
        self._local.rank = rank

    def rank(self):
        return self._local.rank

    def _publish(self, value):
        torch.cuda.synchronize()  # the payload is final before any peer reads it
        self._slots[self.rank()] = value
        self._barrier.wait()
        every = list(self._slots)
        self._barrier.wait()  # everyone has read the slots before they are reused
        return every

    def all_to_all(self, tensor, send_counts, recv_counts):
        chunks = list(torch.split(tensor.contiguous(), list(send_counts), 0))
        every = self._publish(chunks)
        r = self.rank()
        return torch.cat([every[src][r].to(tensor.device) for src in range(self.world)], 0)

    def all_gather(self, tensor):
        return torch.cat([t.to(tensor.device) for t in self._publish(tensor.contiguous().clone())], 0)

    def all_reduce(self, tensor, op="sum"):
        every = self._publish(tensor.clone())
        out = every[0].clone()
        for t in every[1:]:
            out = torch.maximum(out, t) if op == "max" else (torch.minimum(out, t) if op == "min" else out + t)
        tensor.copy_(out)

    def reduce_scatter(self, tensor):
        every = self._publish(tensor.contiguous().clone())
        n = tensor.shape[0] // self.world
        r = self.rank()
        out = every[0][r * n:(r + 1) * n].clone()
        for t in every[1:]:
            out += t[r * n:(r + 1) * n]  # slot (source rank) order, like the fused peer fold
        return out


def _world(group):
    return group.world if isinstance(group, ThreadGroup) else dist.get_world_size(group)


def _rank(group):
    return group.rank() if isinstance(group, ThreadGroup) else dist.get_rank(group)


def _all_reduce(tensor, group, op="sum"):
    if isinstance(group, ThreadGroup):
        return group.all_reduce(tensor, op)
    dop = {"sum": dist.ReduceOp.SUM, "max": dist.ReduceOp.MAX, "min": dist.ReduceOp.MIN}[op]
    dist.all_reduce(tensor, op=dop, group=group)


def _a2a(tensor, send_counts, recv_counts, group):
    """all_to_all_single over dim 0 with per-rank row counts (lists of ints)."""
    if isinstance(group, ThreadGroup):
        return group.all_to_all(tensor, send_counts, recv_counts)
    out = torch.empty((sum(recv_counts),) + tuple(tensor.shape[1:]), dtype=tensor.dtype, device=tensor.device)
    dist.all_to_all_single(out, tensor.contiguous(), recv_counts, send_counts, group=group)
    return out


def _gather_counts(counts, group, host_group=None):
    """Every rank's per-destination counts: matrix[src][dst] (lists), one collective. The counts already live on
    the host, so with `host_group` (a gloo group over the same ranks) they never touch the GPU."""
    world = _world(group)
    if host_group is not None:
        send = torch.tensor(counts, dtype=torch.int64)
        parts = [torch.empty_like(send) for _ in range(world)]
        dist.all_gather(parts, send, group=host_group)
        return torch.stack(parts).tolist()
    send = torch.tensor(counts, dtype=torch.int64, device=_comm_device(group))
    if isinstance(group, ThreadGroup):
        full = group.all_gather(send.view(1, -1))
    else:
        parts = [torch.empty_like(send) for _ in range(world)]
        dist.all_gather(parts, send, group=group)
        full = torch.stack(parts)
    return full.view(world, len(counts)).tolist()


def _comm_device(group):
    if isinstance(group, ThreadGroup) or dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def _all_gather_rows(t, group, world):
    """Rows of every rank's `t`, rank-major, gathered straight into one tensor (no per-rank parts + cat copy)."""
    if isinstance(group, ThreadGroup):
        return group.all_gather(t)
    out = torch.empty((world * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    if world == 1:
        out.copy_(t)
        return out
    dist.all_gather_into_tensor(out, t.contiguous(), group=group)
    return out


def _reduce_scatter_rows(t, group, world, rank):
    if isinstance(group, ThreadGroup):
        return group.reduce_scatter(t)
    if dist.get_backend(group) == "nccl":
        out = torch.empty((t.shape[0] // world,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        dist.reduce_scatter_tensor(out, t.contiguous(), group=group)
        return out
    buf = t.clone()  # gloo: all-reduce then keep this rank's rows
    dist.all_reduce(buf, group=group)
    n = t.shape[0] // world
    return buf[rank * n:(rank + 1) * n].clone()


def _single_node():
    """True when every rank of the job runs on this host (torchrun's LOCAL_WORLD_SIZE == WORLD_SIZE)."""
    lws, ws = os.environ.get("LOCAL_WORLD_SIZE"), os.environ.get("WORLD_SIZE")
    return lws is not None and ws is not None and int(lws) == int(ws)


def _loopback_gloo_group(group, world):
    """A gloo group over the ranks of `group` for the protocol's host-side count exchange, or None.

    Only on a single node: gloo then binds to loopback (its default interface lookup resolves the hostname, which
    may not resolve in a container). GLOO_SOCKET_IFNAME is set only while the group is created and restored
    afterwards, so groups the caller creates later are unaffected; an interface the user chose is kept. Created
    with use_local_synchronization, so only the members of `group` take part (an expert-parallel subgroup of a
    larger job does not deadlock the ranks outside it). Multi-node jobs get None: counts then travel over the
    NCCL group (one device all-gather per exchange)."""
    if world == 1 or not _single_node():
        return None
    ranks = list(range(world)) if group is None else dist.get_process_group_ranks(group)
    prev = os.environ.get("GLOO_SOCKET_IFNAME")
    if prev is None:
        os.environ["GLOO_SOCKET_IFNAME"] = "lo"
    try:
        return dist.new_group(ranks=ranks, backend="gloo", use_local_synchronization=True)
    finally:
        if prev is None:
            os.environ.pop("GLOO_SOCKET_IFNAME", None)


class ShardedLayer:
    """One expert-sharded MEFT layer; ``engine`` does this rank's compute (DeviceEngine on a B200)."""

    def __init__(self, engine, d, M, N, group=None):
        self.eng, self.d, self.M, self.N = engine, d, M, N
        self.group = group
        self.world = _world(group)
        self.rank = _rank(group)
        if N % self.world or M % N:
            raise ValueError("N must be divisible by the world size and M by N")
        self.E, self.N_loc, self.M_loc = M // N, N // self.world, M // self.world
        self.last = {}
        # protocol metadata (per-destination counts) is exchanged host to host over gloo when the data plane is NCCL
        self.host_group = None
        if not isinstance(group, ThreadGroup) and dist.get_backend(group) == "nccl":
            self.host_group = _loopback_gloo_group(group, self.world)
        # Overlap (device engine over NCCL): the bulk all-gathers / reduce-scatters run on their own stream and
        # communicator, so they proceed while the selection exchanges and the FFN compute.
        self.overlap = (isinstance(engine, DeviceEngine) and not isinstance(group, ThreadGroup)
                        and dist.get_backend(group) == "nccl")
        if self.overlap:
            ranks = list(range(self.world)) if group is None else dist.get_process_group_ranks(group)
            self.bulk_group = dist.new_group(ranks=ranks, backend="nccl", use_local_synchronization=True)
            self.comm_stream = torch.cuda.Stream(device=engine.dev)
            # Reduce-scatters of out / grad_h: by default FUSED into the GEMM epilogues over NVLink peer memory
            # (PeerExchange; P > 1 or MEFT_SHARDED_PEER=1), else NCCL on the comm stream with SMs kept free of the
            # persistent FFN GEMMs so its kernels can run beside them (~5% of GEMM throughput).
            env = os.environ.get("MEFT_SHARDED_PEER")
            self.peer_mode = (env == "1") or (env is None and self.world > 1)
            if self.world > 1:  # every rank takes the same path (the peer exchange is collective): MIN over ranks
                flag = torch.tensor([int(self.peer_mode)], dtype=torch.int32,
                                    device="cpu" if self.host_group is not None else engine.dev)
                dist.all_reduce(flag, op=dist.ReduceOp.MIN,
                                group=self.host_group if self.host_group is not None else group)
                self.peer_mode = bool(flag.item())
            self.peer = None
            self.comm_ctx = None
            self.reserve_sms = 0 if (self.peer_mode or self.world == 1) else int(
                os.environ.get("MEFT_SHARDED_RESERVE_SMS", "8"))

    def _peer_exchange(self, T, d):
        """(Re)build the peer receive buffers for T tokens per rank; every rank agrees on success or falls back."""
        if self.peer is not None and self.peer.rows == T:
            return self.peer
        if self.peer is not None:
            self.peer.close()
            self.peer = None
        ok, px = 1, None
        try:
            from .meft import Context
            if self.comm_ctx is None:
                self.comm_ctx = Context(torch.cuda.current_device(), stream=self.comm_stream)
        except Exception:
            ok = 0
        try:  # joins the group's handle exchange even when the context failed (collectives stay matched)
            px = PeerExchange(self.eng.ctx, T, d, group=self.bulk_group, fail_local=not ok)
        except Exception:  # e.g. no CUDA IPC / peer access between these devices, or a failed peer
            ok = 0
        flag = torch.tensor([ok], dtype=torch.int32, device=self.eng.dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=self.bulk_group)
        if int(flag.item()) == 0:
            if px is not None:
                px.close()
            self.peer_mode = False
            self.reserve_sms = 0 if self.world == 1 else int(os.environ.get("MEFT_SHARDED_RESERVE_SMS", "8"))
            return None
        self.peer = px
        return px

    def _barrier(self):  # on the current (comm) stream: every rank's pushed rows have landed
        t = torch.zeros(1, dtype=torch.int32, device=self.eng.dev)
        dist.all_reduce(t, group=self.bulk_group)

    def step(self, h, g, kk, k, lr, g_ready=None):
        """One layer step of this rank's T tokens. g_ready (torch.cuda.Event, optional): g is only final once
        it fires (e.g. an overlapped host->device copy). With the overlapped NCCL path the result carries
        out_ready / grad_h_ready events for copies that should not wait for the whole step."""
        P, r, E = self.world, self.rank, self.E
        eng, grp = self.eng, self.group
        T, d = h.shape
        kk_eff = min(kk, self.N)
        take = min(k, kk_eff * E)
        if self.overlap:  # 8a. all-gather h and g now, behind the whole selection exchange
            cur, cs = torch.cuda.current_stream(), self.comm_stream
            ev_in = torch.cuda.Event()
            ev_in.record(cur)
            ev_h, ev_g = torch.cuda.Event(), torch.cuda.Event()
            with torch.cuda.stream(cs):
                cs.wait_event(ev_in)
                h_all = _all_gather_rows(h, self.bulk_group, P) if P > 1 else h
                ev_h.record(cs)
                if g_ready is not None:
                    cs.wait_event(g_ready)
                g_all = _all_gather_rows(g, self.bulk_group, P) if P > 1 else g
                ev_g.record(cs)
            h.record_stream(cs)
            g.record_stream(cs)
        if not self.overlap:  # h_all is needed by the owners' row gather below
            h_all = _all_gather_rows(h, grp, P)
        # 1. route (exact tau, ascending per token)
        tau = eng.route(h, kk)
        # 2. dispatch (token id, owner-local expert) entries to the expert owners (stable bucket plan on the device);
        # the owners gather the token rows from the all-gathered h they hold anyway -- 8 bytes per entry cross the
        # wire instead of a d-wide bf16 row
        _, send_exp, order, inv, send_counts = eng.dispatch(tau, h, self.N_loc, P, rows=False)
        cmat = _gather_counts(send_counts, grp, self.host_group)  # cmat[src][dst]: rows src dispatches to dst
        recv_counts = [cmat[s][r] for s in range(P)]
        send_ids = (order.long() // kk_eff + r * T).to(torch.int32)
        recv = _a2a(torch.stack([send_ids, send_exp], 1), send_counts, recv_counts, grp)
        recv_ids, recv_exp = recv[:, 0].contiguous(), recv[:, 1].contiguous()
        if self.overlap:
            cur.wait_event(ev_h)  # h_all (the comm stream's all-gather) before the owners read it
            h_all.record_stream(cur)
        recv_rows = eng.gather_rows(h_all, recv_ids)
        # 3-4. owners score; candidate blocks come back in dispatch order
        cand_recv = eng.score(recv_rows, recv_exp)
        cand_back = _a2a(cand_recv, recv_counts, send_counts, grp)
        cand = eng.unpermute(cand_back, order).view(T, kk_eff * E)
        hn, _ = eng.row_stats(h)
        kn_loc, _ = eng.key_stats()
        kn = _all_gather_rows(kn_loc, grp, P)
        # 5. certified classification at the token home
        sure, n_sure, amb, n_amb = eng.classify(cand, tau, hn, kn, take, d)
        # 6. exact re-scoring of the ambiguous candidates by their owners: a request names the owner's receive row
        # of the token's dispatched row (our block starts after the rows of lower source ranks) and the local key
        Ccand = kk_eff * E
        send_off = [sum(send_counts[:o]) for o in range(P)]
        row_base = [sum(cmat[s][o] for s in range(r)) - send_off[o] for o in range(P)]
        req_row, req_key, back, rsend, n_resc = eng.requests(amb, n_amb, tau, inv, E, self.M_loc, P, row_base)
        rmat = _gather_counts(rsend, grp, self.host_group)
        rrecv = [rmat[s][r] for s in range(P)]
        reqs = _a2a(torch.stack([req_row, req_key], 1), rsend, rrecv, grp)  # (receive row, local key) pairs
        in_row, in_key = reqs[:, 0].contiguous(), reqs[:, 1].contiguous()
        x_out = eng.exact(recv_rows, in_row, in_key)
        x_back = _a2a(x_out, rrecv, rsend, grp)
        xs = eng.scatter_exact(x_back, back, T, Ccand)
        # 7. final per-token selection and the global union
        per_token, flags = eng.finalize(sure, n_sure, amb, n_amb, xs, take, self.M)
        union = flags.to(torch.uint8).contiguous()  # the M-entry union bitmap, OR-reduced as a byte max
        _all_reduce(union, grp, "max")
        S = torch.nonzero(union).flatten()
        S_loc = S[(S >= r * self.M_loc) & (S < (r + 1) * self.M_loc)] - r * self.M_loc
        # 8-9. FFN over all tokens on the local part of the union, partial sums back to the homes
        S_loc = S_loc.to(torch.int32).contiguous()
        if self.overlap:
            cur.wait_event(ev_h)  # the forward needs h_all; the backward waits for g_all inside the step
            h_all.record_stream(cur)
            g_all.record_stream(cur)
            timing = bool(os.environ.get("MEFT_SHARDED_EVENT_TIMING"))  # developer probe
            fwd_done, gh_done = torch.cuda.Event(enable_timing=timing), torch.cuda.Event(enable_timing=timing)
            fwd_done.record(cur)  # materialise the CUDA events; the library re-records them
            gh_done.record(cur)
            px = self._peer_exchange(T, d) if self.peer_mode else None
            if self.reserve_sms:
                check(lib().meft_set_gemm_sm_reserve(self.reserve_sms))
            try:
                out_p, gh_p = eng.ffn_local(h_all, g_all, S_loc, lr, g_ready=ev_g, fwd_done=fwd_done,
                                            gh_done=gh_done, peer=px)
            finally:
                if self.reserve_sms:
                    check(lib().meft_set_gemm_sm_reserve(0))
            if px is not None:  # rows were pushed into the homes' buffers by the GEMM epilogues: fold our slots
                ev_o, ev_out = torch.cuda.Event(), torch.cuda.Event()
                with torch.cuda.stream(cs):
                    cs.wait_event(fwd_done)
                    self._barrier()
                    out = px.reduce(self.comm_ctx, 0)
                    ev_o.record(cs)
                    cs.wait_event(gh_done)
                    self._barrier()
                    grad_h = px.reduce(self.comm_ctx, 1)
                    ev_out.record(cs)
                cur.wait_event(ev_out)
                out.record_stream(cur)
                grad_h.record_stream(cur)
            elif P == 1:  # the partial sums are the results: no collective, the library's events mark them final
                out, grad_h, ev_o, ev_out = out_p, gh_p, fwd_done, gh_done
            else:
                ev_o, ev_out = torch.cuda.Event(), torch.cuda.Event()
                with torch.cuda.stream(cs):  # reduce-scatters overlap the backward / weight-gradient GEMMs
                    cs.wait_event(fwd_done)
                    out = _reduce_scatter_rows(out_p, self.bulk_group, P, r)
                    ev_o.record(cs)
                    cs.wait_event(gh_done)
                    grad_h = _reduce_scatter_rows(gh_p, self.bulk_group, P, r)
                    ev_out.record(cs)
                out_p.record_stream(cs)
                gh_p.record_stream(cs)
                cur.wait_event(ev_out)
                out.record_stream(cur)
                grad_h.record_stream(cur)
        else:
            if g_ready is not None:
                torch.cuda.current_stream().wait_event(g_ready)
            g_all = _all_gather_rows(g, grp, P)
            out_p, gh_p = eng.ffn_local(h_all, g_all, S_loc, lr)
            out = _reduce_scatter_rows(out_p, grp, P, r)
            grad_h = _reduce_scatter_rows(gh_p, grp, P, r)
        self.last = dict(union_size=int(S.numel()), local_union=int(S_loc.numel()), rescored=n_resc)
        res = dict(per_token=per_token, tau=tau, unioned=S, out=out, grad_h=grad_h)
        if self.overlap:
            res["out_ready"], res["grad_h_ready"] = ev_o, ev_out
            res["fwd_done"], res["gh_done"] = fwd_done, gh_done
        return res


class CShardedLayer:
    """The same expert-sharded layer step issued entirely inside libmeft_cuda.so (meft_layer_step_sharded, csrc/
    sharded_step.cu): what a C / C++ caller of the drop-in uses. The context's communicator is NCCL, created by the
    library from a unique id that rank 0 broadcasts over `group` (a torch.distributed group), or -- with a
    ThreadGroup -- host callbacks, so a single process can stand in for several ranks on one GPU. Owners gather the
    dispatched token rows from the all-gathered h (no row all-to-all); per-destination counts are all-gathered on
    the device."""

    def __init__(self, ctx, store, w_g, group=None):
        self.ctx, self.store, self.w_g = ctx, store, w_g
        solo = group is None and not dist.is_initialized()  # one rank, no process group: a private communicator
        self.world, self.rank = (1, 0) if solo else (_world(group), _rank(group))
        self._keep = None
        if isinstance(group, ThreadGroup):
            self._set_host_comm(group)
        else:
            uid = (C.c_char * 128)()
            if self.rank == 0:
                check(lib().meft_nccl_unique_id(uid))
            obj = [bytes(uid)]
            if self.world > 1:
                src = 0 if group is None else dist.get_global_rank(group, 0)
                dist.broadcast_object_list(obj, src=src, group=group)
            uid = (C.c_char * 128).from_buffer_copy(obj[0])
            check(lib().meft_ctx_comm_init(ctx.h, uid, self.rank, self.world), ctx.h)

    def _set_host_comm(self, group):
        def all_gather(user, send, nbytes, recv):
            try:
                every = group._publish(C.string_at(send, nbytes))
                C.memmove(recv, b"".join(every), nbytes * len(every))
                return 0
            except Exception:
                return 1

        def all_to_all_v(user, send, send_bytes, recv, recv_bytes):
            try:
                P = group.world
                sizes = [send_bytes[p] for p in range(P)]
                data = C.string_at(send, sum(sizes)) if sum(sizes) else b""
                blocks, o = [], 0
                for n in sizes:
                    blocks.append(data[o:o + n])
                    o += n
                every = group._publish(blocks)
                me = group.rank()
                mine = b"".join(every[src][me] for src in range(P))
                assert len(mine) == sum(recv_bytes[p] for p in range(P))
                if mine:
                    C.memmove(recv, mine, len(mine))
                return 0
            except Exception:
                return 1

        cb = _lib.HostComm(None, _lib.HC_ALL_GATHER(all_gather), _lib.HC_ALL_TO_ALL_V(all_to_all_v))
        self._keep = cb  # the callbacks must outlive the context's use of them
        check(lib().meft_ctx_set_host_comm(self.ctx.h, C.byref(cb), self.rank, self.world), self.ctx.h)

    def close(self):
        lib().meft_ctx_clear_comm(self.ctx.h)

    def step(self, h, g, kk, k, lr, betas=(0.9, 0.999), eps=1e-8, out=None, grad_h=None, want_selection=False):
        """One layer step of this rank's T tokens; returns out / grad_h [T x d] fp32 (and per_token, global ids)."""
        from .meft import selection_shape

        T, d = h.shape
        N = self.w_g.shape[0]
        take, _, _ = selection_shape(self.store.pairs * self.world, N, kk, k)
        out = out if out is not None else torch.empty((T, d), dtype=torch.float32, device=h.device)
        grad_h = grad_h if grad_h is not None else torch.empty_like(out)
        per = torch.empty((T, take), dtype=torch.int32, device=h.device) if want_selection else None
        info = _lib.StepInfo()
        self.ctx.check(lib().meft_layer_step_sharded(self.ctx.h, self.store.h, 0, _p(self.w_g), _p(h), _p(g), T, kk, k,
                                                     betas[0], betas[1], eps, lr, _p(out), _p(grad_h), _p(per),
                                                     C.byref(info)))
        res = {name: getattr(info, name) for name, _ in _lib.StepInfo._fields_}
        peer, overlap = C.c_int(), C.c_int()
        self.ctx.check(lib().meft_ctx_sharded_paths(self.ctx.h, C.byref(peer), C.byref(overlap)))
        # peer_path: partial sums pushed over peer memory; overlap: grad_out all-gathered behind the selection
        res.update(out=out, grad_h=grad_h, peer_path=bool(peer.value), overlap=bool(overlap.value))
        if want_selection:
            res["per_token"] = per
        return res


FULL_TABLE_LIMIT = 24 << 30  # bytes of one global MIXED table set a rank may build to slice its shard from


def make_device_layer(ctx, d, M, N, group=None, seed=1, w_b_seed=0x7001):
    """This rank's shard as a MIXED HBM store: keys from HostStore::init(seed) restricted to the shard (the global
    table is generated once per rank with the reference RNG, then sliced), W_B ~ U(+-1/sqrt d) (torch RNG,
    identical on every rank), router replicated. Layers too large for one GPU (M * d * 28 B above
    FULL_TABLE_LIMIT, e.g. BASELINE config 5's M = 4M: 470 GB) are generated shard by shard instead -- the router
    from the reference stream (replicated), keys and values from torch's device RNG seeded per (seed, rank) -- so
    every rank only ever holds its M/P pairs."""
    from . import meft as G

    P = _world(group)
    r = _rank(group)
    M_loc, N_loc = M // P, N // P
    if M * d * 28 > FULL_TABLE_LIMIT:
        store = G.Store(ctx, 1, d, M_loc, N_loc, G.STORE_MIXED)
        b = 1.0 / math.sqrt(d)
        dev = store.tensor(0, "w_a").device
        gen = torch.Generator(device=dev).manual_seed((seed << 20) + 0x5000 + r)
        for name in ("w_a", "w_b"):
            w, wc = store.tensor(0, name), store.tensor(0, name + "_compute")
            for r0 in range(0, M_loc, 65536):  # chunked: no shard-sized temporaries
                blk = ((torch.rand((min(65536, M_loc - r0), d), generator=gen, device=dev) * 2 - 1) * b).to(
                    torch.bfloat16)
                w[r0:r0 + blk.shape[0]].copy_(blk.float())
                wc[r0:r0 + blk.shape[0]].copy_(blk)
        w_g = torch.from_numpy(G.reference_uniform(seed, 0x5001, (N, d), -b, b, bf16=True)).to(
            device=dev, dtype=torch.bfloat16)
        return DeviceEngine(ctx, store, w_g), store
    full = G.Store(ctx, 1, d, M, N, G.STORE_MIXED)
    full.init_reference(seed)
    store = G.Store(ctx, 1, d, M_loc, N_loc, G.STORE_MIXED)
    for name in ("w_a", "w_a_compute"):
        store.tensor(0, name).copy_(full.tensor(0, name)[r * M_loc:(r + 1) * M_loc])
    gen = torch.Generator(device=store.tensor(0, "w_b").device).manual_seed(w_b_seed)
    b = 1.0 / math.sqrt(d)
    w_b = (torch.rand((M, d), generator=gen, device=gen.device) * 2 - 1) * b
    store.tensor(0, "w_b").copy_(w_b[r * M_loc:(r + 1) * M_loc])
    store.tensor(0, "w_b_compute").copy_(w_b[r * M_loc:(r + 1) * M_loc].to(torch.bfloat16))
    w_g = full.tensor(0, "w_g_compute").clone()
    full.close()
    del w_b
    return DeviceEngine(ctx, store, w_g), store
