#!/usr/bin/env python
"""MEFT adapter layer benchmark (BASELINE.json metric: tokens/sec of fwd + bwd + sparse Adam).

Workload (BASELINE.json configs[1]): LLaMA-7B-shape MEFT layer, d=4096, M=65536 key-value pairs, N=256
experts, K=128 neurons/token, kk=4 experts/token, T=8192 tokens per step, bf16 compute, tables and optimizer
state resident in HBM. One step = meft_ffn (ke_select -> fetch -> sparse FFN) -> sparse_backward ->
scatter_grads -> sparse_adam_update (the reference trainer's per-layer sequence).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload cfg2|cfg1|cfg4]

N>1: one rank per GPU. Launched without torchrun (no WORLD_SIZE in the environment), `--gpus N` re-executes itself
under `torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1` and fails loudly when fewer than N GPUs
are visible. Each rank runs the expert-sharded layer (paper_2406_04984_b200/sharded.py): it owns
N/P experts and M/P pairs and brings T tokens, so the step covers N*T tokens ("scaling": "weak"); tokens,
candidate scores and partial outputs move over NCCL. --sharded runs that path on one GPU too.
Rank 0 prints one JSON line.

Inputs (both arms): HostStore::init(seed 1) tables, W_B ~ U(+-1/sqrt d) from the reference RNG
stream mix_seed(1, 0x7001), h ~ U(-1, 1) from 0x7002, grad_out from 0x7003, all bf16-rounded (the GPU computes in
bf16; the CPU reference gets the same values as doubles).

The reference arm times the UNMODIFIED reference CPU implementation (oracle/_ref, built from /root/reference by
oracle/Makefile) through its public API on all host cores, at the SAME configuration: at N=1 one complete layer
step of the whole T-token batch (meft_ffn -> sparse_backward -> scatter_grads -> sparse_adam_update, |S| = 65,536 at
cfg2; ~580 s on 16 cores, so one step and no warm-up). With --ref-phased (and on rank 0 of N>1 runs) it times a
bounded estimate instead: ke_select + fetch of the whole batch and scatter_grads + sparse_adam_update of its union
measured once, sparse_ffn_pa + sparse_backward measured on slices of the batch's token rows against that same union
and fitted per call as fixed cost + per-row cost (the reference re-transposes the gathered d x |S| tables on every
call), evaluated at T. The GPU arm's `cpu_baseline` is that bounded estimate (a few minutes); the measured complete
step is profiles/r2_reference_full_step.json.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG = dict(lr=1e-4)  # + the chosen WORKLOADS entry (main)
WORKLOADS = {  # BASELINE.json configs[1] (default), [0] (the reference's own CPU workload), [3]
    "cfg2": dict(workload="llama7b_meft_layer", d=4096, pairs=65536, experts=256, k=128, kk=4, tokens=8192),
    "cfg1": dict(workload="reference_cpu_workload", d=512, pairs=4096, experts=64, k=32, kk=4, tokens=256),
    "cfg4": dict(workload="mistral7b_meft_layer_1m", d=4096, pairs=1048576, experts=1024, k=128, kk=4, tokens=8192),
    # the M = 4M corner of the scaling sweep (configs[4]): 470 GB of tables, expert-sharded only (--gpus 8 --strong)
    "cfg5": dict(workload="sweep_m4m_k16", d=4096, pairs=4194304, experts=4096, k=16, kk=4, tokens=8192),
}
METRIC = "MEFT adapter layer tokens/sec (fwd+bwd+sparse update)"
SEED, W_B_STREAM, H_STREAM, G_STREAM = 1, 0x7001, 0x7002, 0x7003


def config_dict(world, sharded=False):
    """The workload as both arms report it (identical dicts: the driver compares the arms on the same config)."""
    per_gpu = CFG["tokens"] // world if CFG.get("strong") else CFG["tokens"]
    return dict(workload=CFG["workload"], d=CFG["d"], pairs=CFG["pairs"], experts=CFG["experts"], k=CFG["k"],
                kk=CFG["kk"], tokens_per_gpu=per_gpu, global_tokens=per_gpu * world,
                parallelism=("single GPU" if world == 1 and not sharded else
                             f"expert-sharded ep{world} (NCCL all-to-all)"),
                inputs="reference RNG streams 0x7001-0x7003 (BASELINE.md §3), bf16-rounded",
                l2=(f"inputs larger than L2 ({CFG['pairs'] * CFG['d'] * 28 / 1e9:.1f} GB of tables per layer)"
                    if CFG["pairs"] * CFG["d"] * 28 > 126e6 else "tables fit in L2 (not flushed; a parity size)"))
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return json.load(f), "measured"
    except OSError:
        return PEAKS_FALLBACK, "fallback"


# ----------------------------------------------------------------------------------------------- clocks

class ClockSampler:
    """Samples SM clock and clock-event reasons via NVML in a background thread during timed regions."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device_index=0, period=0.01):
        self.samples, self.reasons, self.period, self.ok = [], set(), period, False
        self.max_mhz = None
        self.power_mw, self.power_limit_mw = [], None  # board power draw under load vs the enforced cap
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            try:
                self.power_limit_mw = pynvml.nvmlDeviceGetEnforcedPowerLimit(self.h)
            except Exception:
                self.power_limit_mw = None
            self.ok = True
        except Exception:
            self.ok = False
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                try:
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except AttributeError:
                    r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
                try:  # the instantaneous reading (nvmlDeviceGetPowerUsage averages over ~1 s, longer than the
                    # timed region of a short run)
                    fv = nv.nvmlDeviceGetFieldValues(self.h, [nv.NVML_FI_DEV_POWER_INSTANT])[0]
                    self.power_mw.append(fv.value.uiVal if fv.nvmlReturn == 0 else nv.nvmlDeviceGetPowerUsage(self.h))
                except Exception:
                    pass
            except Exception:
                pass
            time.sleep(self.period)

    def start(self):
        if self.ok:
            self._stop.clear()
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        if self._t:
            self._stop.set()
            self._t.join()
            self._t = None

    def summary(self):
        s = sorted(self.samples)
        med = s[len(s) // 2] if s else None
        p = sorted(self.power_mw)
        out = {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(s)}
        if p:  # median board power under load next to the enforced limit (the power cap the GEMMs run into)
            out["power_w"] = round(p[len(p) // 2] / 1e3, 1)
        if self.power_limit_mw:
            out["power_limit_w"] = round(self.power_limit_mw / 1e3, 1)
        return out


# ----------------------------------------------------------------------------------------------- reference arm

def ref_slice_plan(steps):
    """Row counts of the timed reference FFN slices: two sizes (so the per-call fixed cost and the per-row cost
    separate), about 20-45 s of 16-core fp64 work per slice at cfg2; the whole batch at small workloads.
    MEFT_REF_SLICES="16,128" overrides."""
    env = os.environ.get("MEFT_REF_SLICES")
    if env:
        return [int(x) for x in env.split(",")]
    T = CFG["tokens"]
    if T * CFG["pairs"] * CFG["d"] <= 1 << 34:  # small workloads: every slice is the whole batch
        return [T] * max(1, min(steps, 5))
    return [16, 128, 16, 128] if steps > 2 else [16, 128]


def reference_inputs():
    """(store, h, grad_out) of the workload on the reference (oracle/_ref): HostStore::init(seed 1) plus the
    BASELINE.md §3 streams, bf16-rounded -- the values the GPU arm uploads."""
    from oracle import oracle as O
    from paper_2406_04984_b200 import meft as G

    if not O.ref_available():
        O.build()
    d, M, N, T = CFG["d"], CFG["pairs"], CFG["experts"], CFG["tokens"]
    st = O.RefStore(1, d, M, N, seed=SEED)
    b = 1.0 / math.sqrt(d)
    st.set(0, "w_b", G.reference_uniform(SEED, W_B_STREAM, (M, d), -b, b, bf16=True))
    h = G.reference_uniform(SEED, H_STREAM, (T, d), -1.0, 1.0, bf16=True)
    g = G.reference_uniform(SEED, G_STREAM, (T, d), -1.0, 1.0, bf16=True)
    return st, h, g


def run_reference_phased(row_sizes, threads=None):
    """The reference layer step of the full workload through its public API (oracle/ref_capi.cpp ref_step_*):
    ke_select + fetch of the whole batch and scatter_grads + sparse_adam_update of its union timed once; the T x |S|
    FFN forward + backward timed on slices of the batch of the given row counts. Each sparse_backward call pays a
    fixed cost (the reference transposes the two d x |S| gathered tables serially and allocates d x |S| gradients)
    plus a per-row cost, so the full-T call is estimated as fixed + T * per_row, both fitted (least squares) over
    the slices; the composite is labelled as such. Returns a dict (tokens/s, seconds per step, phases, |S|, ...)."""
    import numpy as np

    from oracle import oracle as O

    R = O.ref()
    cores = threads or os.cpu_count()
    R.ref_set_threads(cores)
    st, h, g = reference_inputs()
    T = CFG["tokens"]
    slices, lo = [], 0
    for n in row_sizes:
        n = min(n, T)
        if lo + n > T:
            lo = 0
        slices.append((lo, lo + n))
        lo += n
    t0 = time.perf_counter()
    r = st.step_phases(0, h, g, CFG["kk"], CFG["k"], CFG["lr"], slices)
    wall = time.perf_counter() - t0
    rows = np.array([hi - lo for lo, hi in slices], np.float64)
    fits = {}
    for ph in ("forward", "backward"):
        y = np.array(r[ph], np.float64)
        if len(set(rows.tolist())) >= 2:
            per_row, fixed = np.polyfit(rows, y, 1)
            per_row, fixed = max(per_row, 0.0), max(fixed, 0.0)
        else:  # one slice size: no split, the slice is scaled as a whole
            per_row, fixed = float(np.mean(y / rows)), 0.0
        fits[ph] = (float(fixed), float(per_row))
    phases = dict(select=r["select"], fetch=r["fetch"], scatter=r["scatter"], adam=r["adam"])
    for ph, (fixed, per_row) in fits.items():
        phases[ph] = fixed + per_row * T
    step_s = sum(phases.values())
    return dict(tps=T / step_s, step_s=step_s, phases=phases, union_size=r["union_size"], cores=cores, wall_s=wall,
                slices=[int(x) for x in rows], fits=fits,
                measured={"forward": r["forward"], "backward": r["backward"]})


def run_reference_full(threads=None):
    """One unsliced ref_layer_step of the whole T-token batch (validation of the phased composite)."""
    from oracle import oracle as O

    R = O.ref()
    cores = threads or os.cpu_count()
    R.ref_set_threads(cores)
    st, h, g = reference_inputs()
    t0 = time.perf_counter()
    r = st.layer_step(0, h, g, CFG["kk"], CFG["k"], CFG["lr"], want_outputs=False)
    sec = time.perf_counter() - t0
    phases = dict(zip(["select", "fetch", "forward", "backward", "scatter", "adam"], r["phases"].tolist()))
    return dict(tps=CFG["tokens"] / sec, step_s=sec, phases=phases, union_size=r["union_size"], cores=cores)


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def phased_sample_text(r):
    f_fix, f_row = r["fits"]["forward"]
    b_fix, b_row = r["fits"]["backward"]
    return (f"unmodified reference (oracle/_ref) through its public API, fp64, OpenMP {r['cores']} threads on "
            f"{cpu_model()}, at the full workload (d={CFG['d']} M={CFG['pairs']} N={CFG['experts']} K={CFG['k']} "
            f"kk={CFG['kk']} T={CFG['tokens']}, |S|={r['union_size']} of {CFG['pairs']}): ke_select + fetch of all "
            f"{CFG['tokens']} tokens and scatter_grads + sparse_adam_update of the union measured "
            f"({r['phases']['select']:.1f} + {r['phases']['fetch']:.1f} + {r['phases']['scatter']:.1f} + "
            f"{r['phases']['adam']:.1f} s); sparse_ffn_pa / sparse_backward measured on slices of "
            f"{r['slices']} token rows against that union and fitted per call as fixed + per-row (forward "
            f"{f_fix:.2f} s + {f_row * 1e3:.1f} ms/row, backward {b_fix:.2f} s + {b_row * 1e3:.1f} ms/row), "
            f"evaluated at T={CFG['tokens']}: estimated {r['step_s']:.0f} s per {CFG['tokens']}-token step "
            f"(a measured unsliced step: profiles/r2_reference_full_step.json)")


def reference_arm(args, rank, world):
    if world > 1:  # every rank joins one rendezvous (proves the launch); rank 0 alone runs the CPU reference
        import torch.distributed as dist

        dist.init_process_group("gloo")
        seen = dist.get_world_size()
        dist.barrier()
        if rank != 0:
            dist.destroy_process_group()
            return
    need = 8 * CFG["d"] * CFG["pairs"] * 8  # the reference HostStore: 8 fp64 d x M tables per layer
    try:
        host = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    except (ValueError, OSError):
        host = None
    if host and need > 0.8 * host:
        emit({"impl": "reference", "unavailable": f"the reference's fp64 HostStore needs {need / 1e9:.0f} GB of host "
                                                  f"RAM at {CFG['workload']} (host: {host / 1e9:.0f} GB)"})
        return
    if world == 1 and not args.ref_phased:
        try:
            r = run_reference_full()
        except Exception as e:  # pragma: no cover - surfaced as unavailable, never as a fake number
            emit({"impl": "reference", "unavailable": f"reference CPU run failed: {e}"})
            return
        sample = (f"one complete reference layer step at the workload (meft_ffn -> sparse_backward -> scatter_grads "
                  f"-> sparse_adam_update of all {CFG['tokens']} tokens, |S|={r['union_size']}), unsliced and "
                  f"unextrapolated: fp64, OpenMP {r['cores']} threads on {cpu_model()}; one step because a step "
                  f"takes ~10 min on 16 cores (--steps / --warmup apply to the GPU arm; --ref-phased times the "
                  f"bounded phased estimate instead)")
        value, ms, steps_done = r["tps"], r["step_s"] * 1e3, 1
        args.warmup = 0
    else:
        try:
            r = run_reference_phased(ref_slice_plan(args.steps))
        except Exception as e:  # pragma: no cover
            emit({"impl": "reference", "unavailable": f"reference CPU run failed: {e}"})
            return
        sample = phased_sample_text(r)
        value, ms, steps_done = r["tps"], r["step_s"] * 1e3, len(r["slices"])
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": steps_done, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if CFG.get("strong") else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config_dict(world),
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": r["cores"], "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "phase_seconds": r["phases"], "union_size": r["union_size"],
    }
    if world > 1:
        line["ranks_joined"] = seen
        import torch.distributed as dist

        dist.destroy_process_group()
    emit(line)


# ----------------------------------------------------------------------------------------------- our arm

def our_arm(args, rank, world, local_rank):
    import torch

    from paper_2406_04984_b200 import meft as G

    dist = torch.distributed if world > 1 else None  # barriers / max-over-ranks only with several ranks
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    d, M, N, K, kk, T, lr = (CFG[x] for x in ("d", "pairs", "experts", "k", "kk", "tokens", "lr"))
    if CFG.get("strong"):
        if T % world:
            raise SystemExit(f"bench.py: --strong needs the workload's {T} tokens divisible by {world} ranks")
        T //= world  # strong scaling: the global batch is split over the ranks
    if M * d * 28 > 170e9 and world == 1 and not args.sharded:
        raise SystemExit(f"bench.py: {CFG['workload']} needs {M * d * 28 / 1e9:.0f} GB of tables: expert-shard it "
                         "(--gpus N, N >= 4 for M = 4M)")

    if torch.cuda.device_count() < world or not torch.cuda.is_available():
        raise SystemExit(f"bench.py: {world} rank(s) need {world} visible GPUs, found {torch.cuda.device_count()}")
    ctx = G.Context(local_rank)
    # BASELINE.md §3 inputs from the reference RNG streams (rank r of a sharded run: stream + 0x100 * r), bf16
    h = torch.from_numpy(G.reference_uniform(SEED, H_STREAM + 0x100 * rank, (T, d), -1.0, 1.0, bf16=True)).to(
        device=dev, dtype=torch.bfloat16)
    g = torch.from_numpy(G.reference_uniform(SEED, G_STREAM + 0x100 * rank, (T, d), -1.0, 1.0, bf16=True)).to(
        device=dev, dtype=torch.bfloat16)
    out = torch.empty((T, d), dtype=torch.float32, device=dev)
    grad_h = torch.empty((T, d), dtype=torch.float32, device=dev)
    sharded = world > 1 or args.sharded
    if not sharded:
        store = G.Store(ctx, 1, d, M, N, G.STORE_COMPACT if args.precision == "compact" else G.STORE_MIXED)
        store.init_reference(seed=SEED)  # HostStore::init tables (reference RNG streams 0x5000/0x5001)
        b = 1.0 / math.sqrt(d)
        if M * d <= 1 << 28:  # W_B ~ U(+-1/sqrt d) from stream 0x7001, bf16-rounded
            store.upload(0, "w_b", G.reference_uniform(SEED, W_B_STREAM, (M, d), -b, b, bf16=True))
        else:  # cfg4 (M = 1M: 34 GB of host doubles): the same distribution from torch's device RNG, in chunks
            wgen = torch.Generator(device=dev).manual_seed(W_B_STREAM)
            w_b, w_bc = store.tensor(0, "w_b"), store.tensor(0, "w_b_compute")
            for r0 in range(0, M, 65536):
                blk = ((torch.rand((min(65536, M - r0), d), generator=wgen, device=dev) * 2 - 1) * b).to(
                    torch.bfloat16)
                w_b[r0:r0 + blk.shape[0]].copy_(blk.float())
                w_bc[r0:r0 + blk.shape[0]].copy_(blk)
            del blk

        base = None
        if args.base_ffn:  # the frozen base FFN of the layer too (optional n = 11008 run)
            bgen = torch.Generator(device=dev).manual_seed(0x7004)
            w_in = ((torch.rand((d, args.base_ffn), generator=bgen, device=dev) * 2 - 1) / math.sqrt(d)).to(torch.bfloat16)
            w_out = ((torch.rand((args.base_ffn, d), generator=bgen, device=dev) * 2 - 1)
                     / math.sqrt(args.base_ffn)).to(torch.bfloat16)
            base = (w_in, w_out, 0)

        def step():
            return store.layer_step(0, h, g, kk, K, lr, out=out, grad_h=grad_h, base=base)
    else:
        # expert-sharded layer: this rank owns N/P experts and M/P pairs; tokens are exchanged over NCCL
        from paper_2406_04984_b200 import sharded as SH

        eng, store = SH.make_device_layer(ctx, d, M, N, seed=1)
        if args.sharded_impl == "capi":  # the whole protocol inside libmeft_cuda.so (meft_layer_step_sharded)
            layer = SH.CShardedLayer(ctx, store, eng.w_g, group=torch.distributed.group.WORLD)

            def step():
                l0 = G.kernel_launches()
                res = layer.step(h, g, kk, K, lr, out=out, grad_h=grad_h)
                return dict(union_size=res["union_size"], rescored=res["rescored"], fallbacks=0,
                            gpu_launches=G.kernel_launches() - l0)
        else:  # the Python orchestration over the C ABI's blocks (comm-stream overlap, fused peer reduce-scatter)
            layer = SH.ShardedLayer(eng, d, M, N)

            def step():
                l0 = G.kernel_launches()
                res = layer.step(h, g, kk, K, lr)
                out.copy_(res["out"])
                grad_h.copy_(res["grad_h"])
                info = dict(layer.last)
                info["gpu_launches"] = G.kernel_launches() - l0
                info["fallbacks"] = 0
                return info

    for _ in range(args.warmup):
        info = step()
    torch.cuda.synchronize()
    ctx.read_timing()  # drop warm-up records
    ctx.set_timing(True)

    clocks = ClockSampler(local_rank)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    ev0.record()
    launches = 0
    usizes = []
    rescored = fallbacks = 0
    for _ in range(args.steps):
        info = step()
        launches += info["gpu_launches"]
        usizes.append(info["union_size"])
        rescored += info["rescored"]
        fallbacks += info["fallbacks"]
    ev1.record()
    torch.cuda.synchronize()
    clocks.stop()
    if dist:
        dist.barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    phases = ctx.read_timing()
    ctx.set_timing(False)
    if dist:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * T / (ms * 1e-3)

    # ---- end to end through the C-ABI host entry point (pinned host buffers, copies inside the timed region)
    h_host = h.cpu().pin_memory()
    g_host = g.cpu().pin_memory()
    out_host = torch.empty((T, d), dtype=torch.float32).pin_memory()
    gh_host = torch.empty((T, d), dtype=torch.float32).pin_memory()
    e2e_steps = max(3, min(args.steps, 10))
    copy_stream = torch.cuda.Stream(device=dev)
    g_ev = torch.cuda.Event()

    def e2e_step():
        if not sharded:  # one C-ABI call: copies overlapped with the step inside meft_layer_step_host
            store.layer_step_host(0, h_host, g_host, kk, K, lr, out_host, gh_host)
        elif args.sharded_impl == "capi":  # copies in, one C-ABI call, copies out
            h.copy_(h_host, non_blocking=True)
            g.copy_(g_host, non_blocking=True)
            layer.step(h, g, kk, K, lr, out=out, grad_h=grad_h)
            out_host.copy_(out, non_blocking=True)
            gh_host.copy_(grad_h, non_blocking=True)
            torch.cuda.synchronize()
        else:  # h first; g, out and grad_h move on a copy stream while the step computes
            h.copy_(h_host, non_blocking=True)
            with torch.cuda.stream(copy_stream):
                g.copy_(g_host, non_blocking=True)
                g_ev.record(copy_stream)
            res = layer.step(h, g, kk, K, lr, g_ready=g_ev)
            ready = [res.get("out_ready"), res.get("grad_h_ready")]
            for dst, src, ev in ((out_host, res["out"], ready[0]), (gh_host, res["grad_h"], ready[1])):
                if ev is not None:
                    copy_stream.wait_event(ev)
                else:
                    copy_stream.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(copy_stream):
                    dst.copy_(src, non_blocking=True)
                src.record_stream(copy_stream)
            torch.cuda.synchronize()

    e2e_step()
    if dist:
        dist.barrier()
    clocks.start()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    clocks.stop()
    if dist:
        t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = world * T / e2e_s

    if rank != 0:
        return

    # ---- roofline of the dominant kernel (tcgen05 GEMM) from live CUDA-event phase timings
    peaks, peak_src = load_peaks()
    S = sum(usizes) / len(usizes)
    gemm_ms = (phases["ffn_forward"][0] + phases["ffn_backward"][0]) / args.steps
    gemm_launches = 6  # z, out | dA, gW_B, gW_A, grad_h per step (the phases also hold two ~us run-table kernels)
    gemm_flops = 2.0 * T * d * S  # algorithmic flops of one of the six T x d x |S| GEMMs
    gemm_tflops = gemm_flops / (gemm_ms / gemm_launches * 1e-3) / 1e12
    tc_peak = peaks.get("bf16_tflops_sustained", PEAKS_FALLBACK["bf16_tflops_sustained"])
    hbm = peaks.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"])
    # sparse Adam: fused into the two grad-W GEMM epilogues by default (the gradient never reaches HBM: read w,m,v
    # + write w,m,v fp32 + bf16 copy = 26 B/entry); MEFT_ADAM_EPILOGUE=0 runs the separate pass over a gradient
    # block (+ the gradient read: 30 B/entry)
    adam_fused = os.environ.get("MEFT_ADAM_EPILOGUE", "1") != "0"
    per_entry = (26.0 if adam_fused else 30.0) - (8.0 if args.precision == "compact" else 0.0)  # bf16 m, v: -8 B
    adam_bytes = 2 * S * d * per_entry  # key and value rows
    gather_bytes = 2 * S * d * 2 * 2.0
    adam_ms = phases["adam"][0] / args.steps
    gather_ms = phases["gather"][0] / args.steps
    select_ms = phases["select"][0] / args.steps
    bwd_ms = phases["ffn_backward"][0] / args.steps
    # composite layer roofline: sum_k max(F_k / TC peak, B_k / HBM peak); with the fused Adam each
    # grad-W GEMM is one kernel moving its operands plus half the Adam bytes under its flops
    gemm_t = gemm_flops / (tc_peak * 1e12)
    if adam_fused:
        adam_gemm_t = max(gemm_t, (adam_bytes / 2 + (T * S + T * d) * 2.0) / (hbm * 1e9))
        ffn_roof = 4 * gemm_t + 2 * adam_gemm_t
    else:
        ffn_roof = 6 * gemm_t + adam_bytes / (hbm * 1e9)
    key_bytes = (M * d * 2) + T * d * 2
    roof_ms = (ffn_roof + key_bytes / (hbm * 1e9) + 2 * T * N * d / (tc_peak * 1e12)) * 1e3

    # DRAM traffic per GEMM launch from the committed ncu --set full capture of one step's six GEMMs
    traffic = None  # the committed capture is of the cfg2 step only
    tpath = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "gemm_traffic.json")
    if os.path.exists(tpath) and CFG["workload"] == "llama7b_meft_layer":
        with open(tpath) as f:
            traffic = json.load(f).get("mean_dram_bytes_per_launch")

    cpu = None
    if world == 1 and not args.skip_cpu_baseline and not args.base_ffn:
        try:  # the reference arm's phased measurement on a bounded sample: two slice sizes
            r = run_reference_phased(ref_slice_plan(2))
            cpu = {"value": r["tps"], "unit": "tokens/s", "cores": r["cores"], "kind": "reference",
                   "sample": phased_sample_text(r), "phase_seconds": r["phases"]}
        except Exception as e:
            cpu = {"value": None, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"not run: {e}"}

    line = {
        "metric": METRIC,
        "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong" if CFG.get("strong") else "weak",
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (HostStore::init tables; W_B, h, grad_out from the reference RNG streams, bf16)",
        "config": config_dict(world, sharded),
        "precision": "bf16 compute, fp32 master weights, " + ("bf16 Adam moments (COMPACT)" if args.precision ==
                                                                  "compact" else "fp32 Adam moments"),
        "union_size": S, "base_ffn": args.base_ffn,
        "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": 2 * T * d * 2,
                "d2h_bytes_per_step": 2 * T * d * 4, "ms_per_step": e2e_s * 1e3,
                "path": "meft_layer_step_host (C ABI, pinned host buffers)" if not sharded else
                        "sharded layer step with pinned host copies in and out"},
        "roofline": {"bound": "tensor",
                     "kernel": "k_gemm_bf16_pair (tcgen05 cta_group::2 FFN GEMM, 6 per step"
                               + ("; the two grad-W launches also run the sparse Adam in their epilogue)"
                                  if adam_fused else ")"),
                     "achieved": gemm_tflops,
                     "peak": tc_peak, "unit": "TFLOP/s", "frac": gemm_tflops / tc_peak, "traffic": traffic,
                     "traffic_unit": "bytes per launch (ncu dram read+write, profiles/gemm_traffic.json)",
                     "peak_source": f"{peak_src} bf16_tflops_sustained",
                     "per_launch": {"flops": gemm_flops, "ms": gemm_ms / gemm_launches}},
        "layer_roofline": {"roofline_ms": roof_ms, "measured_ms": ms, "frac": roof_ms / ms},
        "phases_ms": {"select": select_ms, "gather": gather_ms, "ffn_forward": phases["ffn_forward"][0] / args.steps,
                      "ffn_backward": phases["ffn_backward"][0] / args.steps, "adam": adam_ms},
        "hbm_kernels": {"adam_placement": "grad-W GEMM epilogues" if adam_fused else "separate pass",
                        "adam_bytes_per_step": adam_bytes,
                        "adam_gbs": adam_bytes / (adam_ms * 1e-3) / 1e9 if adam_ms and not adam_fused else None,
                        "gather_gbs": gather_bytes / (gather_ms * 1e-3) / 1e9 if gather_ms else None,
                        "peak_gbs": hbm},
        "selection": {"algorithm": "certified tcgen05 scoring + exact fp64 re-scoring (bit-exact indices)",
                      "rescored_per_token": rescored / (args.steps * T),
                      "sequential_fallbacks_per_step": fallbacks / args.steps},
        "cpu_baseline": cpu,
        "clocks": clocks.summary(),
        "gpu_launches": launches,
    }
    emit(line)


# The JSON line is the only thing on stdout: everything else written to fd 1 (NCCL's version banner, library
# prints) is redirected to stderr, and the line goes to a saved copy of the original stdout.
_JSON_OUT = None


def _claim_stdout():
    global _JSON_OUT
    if _JSON_OUT is None:
        sys.stdout.flush()
        _JSON_OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)


def emit(line):
    _claim_stdout()
    _JSON_OUT.write(json.dumps(line) + "\n")
    _JSON_OUT.flush()


def _free_port():
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def spawn_ranks(n):
    """`--gpus N` without a launcher: re-execute this command under torch.distributed.run with N local ranks
    (rendezvous on 127.0.0.1). Rank 0's JSON line reaches our stdout; the exit code is the launcher's."""
    import subprocess

    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    print(f"bench.py: launching {n} ranks: {' '.join(cmd)}", file=sys.stderr)
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--skip-cpu-baseline", action="store_true")
    ap.add_argument("--ref-phased", action="store_true",
                    help="reference arm: the bounded phased estimate (slices of the batch, per-call fixed cost + "
                         "per-row cost fitted) instead of one complete T-token reference step (~10 min at cfg2)")
    ap.add_argument("--sharded", action="store_true", help="run the expert-sharded layer even on one GPU")
    ap.add_argument("--sharded-impl", choices=["python", "capi"], default="python",
                    help="expert-sharded step: Python orchestration (overlapped, fused peer reduce-scatter) or the "
                         "C-ABI meft_layer_step_sharded")
    ap.add_argument("--base-ffn", type=int, default=0,
                    help="also run the frozen base FFN of width n (SiLU), e.g. 11008 for LLaMA-7B (single GPU)")
    ap.add_argument("--precision", choices=["mixed", "compact"], default="mixed",
                    help="store precision: fp32 Adam moments (default) or bf16 moments (COMPACT, opt-in)")
    ap.add_argument("--strong", action="store_true",
                    help="strong scaling: the workload's T tokens are split over the ranks (default: weak, T per rank)")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="cfg2",
                    help="cfg2: the LLaMA-7B-shape layer (default, BASELINE configs[1]); cfg1: the reference's own "
                         "CPU workload (configs[0]); cfg4: the Mistral-7B shape with M = 1,048,576 neurons and "
                         "1,024 experts (configs[3], meant for --gpus 8)")
    args = ap.parse_args()
    CFG.update(WORKLOADS[args.workload])
    CFG["strong"] = args.strong
    args.warmup = max(args.warmup, 0)
    if args.gpus < 1:
        raise SystemExit("bench.py: --gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        if args.impl == "ours":
            import torch

            if torch.cuda.device_count() < args.gpus:
                raise SystemExit(f"bench.py: --gpus {args.gpus} but only {torch.cuda.device_count()} GPU(s) visible")
        sys.exit(spawn_ranks(args.gpus))
    _claim_stdout()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: launched with WORLD_SIZE={world} but --gpus {args.gpus}")
    if args.impl == "reference":
        reference_arm(args, rank, world)
        return
    distributed = world > 1 or args.sharded
    if distributed:
        import torch

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(_free_port()))
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        our_arm(args, rank, world, local_rank)
    finally:
        if distributed:
            import torch

            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
