"""Sustained run of the cfg2 layer step (one B200): N minutes of back-to-back steps with the reference's
check_finite on (meft_ctx_set_check_finite: every step scans out / grad_h for NaN / Inf), reporting per-window step
time, union size, SM clock and board power -- does the power-capped rate hold, and do the tables stay finite?

  python tools/soak.py [minutes=3]
"""
import json
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_04984_b200 import meft as G  # noqa: E402


def main():
    minutes = float(sys.argv[1]) if len(sys.argv) > 1 else 3.0
    import pynvml as nv

    nv.nvmlInit()
    hdl = nv.nvmlDeviceGetHandleByIndex(0)
    d, M, N, K, kk, T = 4096, 65536, 256, 128, 4, 8192
    ctx = G.Context(0)
    ctx.set_check_finite(True)
    st = G.Store(ctx, 1, d, M, N, G.STORE_MIXED)
    b = 1.0 / d ** 0.5
    gen = torch.Generator(device="cuda").manual_seed(1)
    with torch.no_grad():
        for name in ("w_a", "w_b", "w_g"):
            w = st.tensor(0, name)
            w.uniform_(-b, b, generator=gen)
            st.tensor(0, name + "_compute").copy_(w.to(torch.bfloat16))
    # a few distinct batches, cycled (the selection and the union move with the inputs and the updated tables)
    batches = [((torch.rand((T, d), generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16),
                (torch.rand((T, d), generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16)) for _ in range(4)]
    out = torch.empty((T, d), device="cuda")
    gh = torch.empty_like(out)
    samples, stop = [], threading.Event()

    def sample():
        while not stop.is_set():
            try:
                fv = nv.nvmlDeviceGetFieldValues(hdl, [nv.NVML_FI_DEV_POWER_INSTANT])[0]
                samples.append((time.perf_counter(), nv.nvmlDeviceGetClockInfo(hdl, nv.NVML_CLOCK_SM),
                                fv.value.uiVal / 1e3, nv.nvmlDeviceGetTemperature(hdl, nv.NVML_TEMPERATURE_GPU)))
            except Exception:
                pass
            time.sleep(0.02)

    th = threading.Thread(target=sample, daemon=True)
    th.start()
    t0 = time.perf_counter()
    step, window = 0, 200
    lines = []
    while time.perf_counter() - t0 < minutes * 60:
        w0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sizes = []
        for i in range(window):
            h, g = batches[(step + i) % len(batches)]
            r = st.layer_step(0, h, g, kk, K, 1e-4, out=out, grad_h=gh)  # raises on a non-finite out / grad_h
            sizes.append(r["union_size"])
        e1.record()
        torch.cuda.synchronize()
        step += window
        w1 = time.perf_counter()
        ws = [s for s in samples if w0 <= s[0] <= w1]
        med = lambda xs: sorted(xs)[len(xs) // 2] if xs else None  # noqa: E731
        line = {"steps_done": step, "elapsed_s": round(w1 - t0, 1), "ms_per_step": e0.elapsed_time(e1) / window,
                "union_min": min(sizes), "union_max": max(sizes), "sm_mhz": med([s[1] for s in ws]),
                "power_w": med([s[2] for s in ws]), "temp_c": med([s[3] for s in ws])}
        lines.append(line)
        print(json.dumps(line), flush=True)
    stop.set()
    th.join()
    w = [float(torch.isfinite(st.tensor(0, n)).all()) for n in ("w_a", "w_b", "m_a", "v_a", "m_b", "v_b")]
    ms = [l["ms_per_step"] for l in lines]
    print(json.dumps({"summary": True, "steps": step, "minutes": minutes, "tables_finite": all(w),
                      "ms_per_step_first_window": ms[0], "ms_per_step_last_window": ms[-1],
                      "ms_per_step_min": min(ms), "ms_per_step_max": max(ms),
                      "max_pair_step": int(st.tensor(0, "pair_step").max())}))


if __name__ == "__main__":
    main()
