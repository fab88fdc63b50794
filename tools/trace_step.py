"""Developer harness: GPU timeline of fused cfg2 layer steps via torch.profiler (CUPTI kernel records), printing
each kernel's start offset, duration and the idle gap before it -- launch gaps and host syncs show up as gaps.
   python tools/trace_step.py [steps]"""
import json
import os
import sys
import tempfile

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from profile_step import make_step  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    step = make_step()
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            step()
        torch.cuda.synchronize()
    path = os.path.join(tempfile.mkdtemp(), "trace.json")
    prof.export_chrome_trace(path)
    ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
    ev.sort(key=lambda e: e["ts"])
    t0, prev_end = ev[0]["ts"], ev[0]["ts"]
    busy = 0.0
    for e in ev:
        gap = e["ts"] - prev_end
        busy += e["dur"]
        print(f"{e['ts'] - t0:10.1f} {e['dur']:9.1f} gap {gap:7.1f}  {e['name'][:80]}")
        prev_end = max(prev_end, e["ts"] + e["dur"])
    span = prev_end - t0
    print(f"span {span:.1f} us, kernels busy {busy:.1f} us, idle {span - busy:.1f} us over {steps} steps")


if __name__ == "__main__":
    main()
