"""Board power and SM clock while the cfg2 layer step runs back to back (one B200), sampled through NVML every
~5 ms: the instantaneous and averaged power readings, the enforced limit, the SM clock and the clock-event
reasons -- the evidence behind "the GEMMs run into the board's power cap".

  python tools/power_probe.py [seconds=6] [mixed|compact]
"""
import json
import os
import statistics
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_04984_b200 import meft as G  # noqa: E402


def sampler(h, nv, stop, out):
    fields = [nv.NVML_FI_DEV_POWER_INSTANT, nv.NVML_FI_DEV_POWER_AVERAGE]
    while not stop.is_set():
        row = {"t": time.perf_counter(), "sm_mhz": nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
               "usage_w": nv.nvmlDeviceGetPowerUsage(h) / 1e3}
        try:
            vals = nv.nvmlDeviceGetFieldValues(h, fields)
            row["instant_w"] = vals[0].value.uiVal / 1e3 if vals[0].nvmlReturn == 0 else None
            row["average_w"] = vals[1].value.uiVal / 1e3 if vals[1].nvmlReturn == 0 else None
        except Exception:
            pass
        try:
            row["reasons"] = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        except Exception:
            row["reasons"] = None
        out.append(row)
        time.sleep(0.005)


def summarise(rows, name):
    res = {"phase": name, "samples": len(rows)}
    for k in ("sm_mhz", "usage_w", "instant_w", "average_w"):
        v = sorted(r[k] for r in rows if r.get(k) is not None)
        if v:
            res[k] = {"p10": v[len(v) // 10], "median": v[len(v) // 2], "p90": v[9 * len(v) // 10], "max": v[-1]}
    bits = [r["reasons"] for r in rows if r.get("reasons") is not None]
    if bits:
        res["sw_power_cap_fraction"] = sum(1 for b in bits if b & 0x4) / len(bits)
    return res


def main():
    seconds = float(sys.argv[1]) if len(sys.argv) > 1 else 6.0
    prec = sys.argv[2] if len(sys.argv) > 2 else "mixed"
    import pynvml as nv

    nv.nvmlInit()
    h = nv.nvmlDeviceGetHandleByIndex(0)
    d, M, N, K, kk, T = 4096, 65536, 256, 128, 4, 8192
    ctx = G.Context(0)
    st = G.Store(ctx, 1, d, M, N, G.STORE_COMPACT if prec == "compact" else G.STORE_MIXED)
    b = 1.0 / d ** 0.5
    gen = torch.Generator(device="cuda").manual_seed(1)
    with torch.no_grad():
        for name in ("w_a", "w_b", "w_g"):
            w = st.tensor(0, name)
            w.uniform_(-b, b, generator=gen)
            st.tensor(0, name + "_compute").copy_(w.to(torch.bfloat16))
    hh = (torch.rand((T, d), generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16)
    gg = (torch.rand((T, d), generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16)
    out = torch.empty((T, d), device="cuda")
    gh = torch.empty_like(out)
    for _ in range(3):
        st.layer_step(0, hh, gg, kk, K, 1e-4, out=out, grad_h=gh, want_info=False)
    torch.cuda.synchronize()

    rows, stop = [], threading.Event()
    th = threading.Thread(target=sampler, args=(h, nv, stop, rows), daemon=True)
    th.start()
    time.sleep(1.0)  # idle
    t_load = time.perf_counter()
    steps = 0
    while time.perf_counter() - t_load < seconds:
        for _ in range(10):
            st.layer_step(0, hh, gg, kk, K, 1e-4, out=out, grad_h=gh, want_info=False)
        torch.cuda.synchronize()
        steps += 10
    t_end = time.perf_counter()
    time.sleep(0.5)
    stop.set()
    th.join()
    limit = nv.nvmlDeviceGetEnforcedPowerLimit(h) / 1e3
    idle = [r for r in rows if r["t"] < t_load - 0.1]
    load = [r for r in rows if t_load + 1.0 < r["t"] < t_end]  # skip the first second (the 1-s average settles)
    print(json.dumps({"precision": prec, "enforced_limit_w": limit, "steps": steps,
                      "ms_per_step": (t_end - t_load) * 1e3 / steps,
                      "idle": summarise(idle, "idle"), "load": summarise(load, "load")}))


if __name__ == "__main__":
    main()
