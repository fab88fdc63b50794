"""Developer harness: GPU timeline of fused cfg2 layer steps via torch.profiler (CUPTI kernel records), printing
each kernel's start offset, duration and the idle gap before it -- launch gaps and host syncs show up as gaps.
   python tools/trace_step.py [steps] [sharded]     (sharded: the expert-sharded layer at world size 1 over NCCL)"""
import json
import os
import sys
import tempfile

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from profile_step import make_step  # noqa: E402


def make_sharded_step():
    import torch.distributed as dist

    from paper_2406_04984_b200 import meft as G
    from paper_2406_04984_b200 import sharded as SH

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    d, M, N, K, kk, T = 4096, 65536, 256, 128, 4, 8192
    ctx = G.Context(0)
    eng, _ = SH.make_device_layer(ctx, d, M, N, seed=1)
    layer = SH.ShardedLayer(eng, d, M, N)
    gen = torch.Generator(device="cuda").manual_seed(0x7002)
    h = (torch.rand((T, d), generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16)
    g = (torch.rand((T, d), generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16)
    return lambda: layer.step(h, g, kk, K, 1e-4)


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    step = make_sharded_step() if len(sys.argv) > 2 and sys.argv[2] == "sharded" else make_step()
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    acts = [ProfilerActivity.CUDA] + ([ProfilerActivity.CPU] if os.environ.get("TRACE_CPU") else [])
    with profile(activities=acts) as prof:
        for _ in range(steps):
            step()
        torch.cuda.synchronize()
    path = os.path.join(tempfile.mkdtemp(), "trace.json")
    prof.export_chrome_trace(path)
    allev = json.load(open(path))["traceEvents"]
    if os.environ.get("TRACE_CPU"):  # host-side ops longer than 40 us (python_function / cpu_op / user_annotation)
        cpu = sorted([e for e in allev if e.get("cat") in ("cpu_op", "python_function") and e.get("dur", 0) > 40],
                     key=lambda e: e["ts"])
        c0 = cpu[0]["ts"] if cpu else 0
        for e in cpu:
            print(f"CPU {e['ts'] - c0:10.1f} {e['dur']:9.1f}  {e['name'][:90]}")
    ev = [e for e in allev if e.get("cat") == "kernel"]
    ev.sort(key=lambda e: e["ts"])
    t0, prev_end = ev[0]["ts"], ev[0]["ts"]
    busy = 0.0
    for e in ev:
        gap = e["ts"] - prev_end
        busy += e["dur"]
        if e["dur"] > 20 or gap > 20 or os.environ.get("TRACE_ALL"):
            print(f"{e['ts'] - t0:10.1f} {e['dur']:9.1f} gap {gap:7.1f}  {e['name'][:80]}")
        prev_end = max(prev_end, e["ts"] + e["dur"])
    span = prev_end - t0
    print(f"span {span:.1f} us, kernels busy {busy:.1f} us, idle {span - busy:.1f} us over {steps} steps")


if __name__ == "__main__":
    main()
