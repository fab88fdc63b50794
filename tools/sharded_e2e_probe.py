"""Developer probe: which host<->device copy of the sharded layer step is left exposed (world size 1, NCCL).
Times the step alone and with each copy added, wall clock around synchronised steps."""
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_04984_b200 import meft as G  # noqa: E402
from paper_2406_04984_b200 import sharded as SH  # noqa: E402


def main():
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29561")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    d, M, N, K, kk, T = 4096, 65536, 256, 128, 4, 8192
    if os.environ.get("PROBE_MAIN_STREAM"):  # run everything on a non-default (non-blocking) stream
        torch.cuda.set_stream(torch.cuda.Stream())
    ctx = G.Context(0)
    eng, _ = SH.make_device_layer(ctx, d, M, N, seed=1)
    layer = SH.ShardedLayer(eng, d, M, N)
    h = (torch.rand((T, d), device="cuda") * 2 - 1).to(torch.bfloat16)
    g = (torch.rand((T, d), device="cuda") * 2 - 1).to(torch.bfloat16)
    hh, gh = h.cpu().pin_memory(), g.cpu().pin_memory()
    oh = torch.empty((T, d), dtype=torch.float32).pin_memory()
    ghh = torch.empty_like(oh).pin_memory()
    cs = torch.cuda.Stream()
    gev = torch.cuda.Event()

    def run(h2d_h, h2d_g, d2h):
        if h2d_h:
            h.copy_(hh, non_blocking=True)
        if h2d_g:
            with torch.cuda.stream(cs):
                g.copy_(gh, non_blocking=True)
                gev.record(cs)
        res = layer.step(h, g, kk, K, 1e-4, g_ready=gev if h2d_g else None)
        if d2h:
            for dst, src, ev in ((oh, res["out"], res.get("out_ready")), (ghh, res["grad_h"], res.get("grad_h_ready"))):
                cs.wait_event(ev)
                with torch.cuda.stream(cs):
                    dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()

    # when do the results become final, relative to the step start?
    for _ in range(3):
        t0, to, tg, te = (torch.cuda.Event(enable_timing=True) for _ in range(4))
        t0.record()
        res = layer.step(h, g, kk, K, 1e-4)
        cs.wait_event(res["out_ready"])
        to.record(cs)
        cs.wait_event(res["grad_h_ready"])
        tg.record(cs)
        te.record()
        torch.cuda.synchronize()
        print(f"out_ready {t0.elapsed_time(to):7.2f}  grad_h_ready {t0.elapsed_time(tg):7.2f}  step end "
              f"{t0.elapsed_time(te):7.2f} ms", flush=True)
        if os.environ.get("MEFT_SHARDED_EVENT_TIMING"):
            print(f"   library fwd_done {t0.elapsed_time(res['fwd_done']):7.2f}  gh_done "
                  f"{t0.elapsed_time(res['gh_done']):7.2f}", flush=True)
    for name, args in (("step", (0, 0, 0)), ("+h", (1, 0, 0)), ("+g", (0, 1, 0)), ("+d2h", (0, 0, 1)),
                       ("all", (1, 1, 1)), ("step", (0, 0, 0))):
        for _ in range(2):
            run(*args)
        t0 = time.perf_counter()
        for _ in range(5):
            run(*args)
        print(f"{name:6s} {(time.perf_counter() - t0) / 5 * 1e3:8.2f} ms", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
