"""bench.py's output contract (the driver parses exactly one JSON line on stdout): the reference arm on CPU with a
tiny bounded sample, and the GPU arm's keys (roofline, cpu_baseline, e2e, clocks, gpu_launches) on a B200."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None, timeout=900):
    e = dict(os.environ)
    e.update(env or {})
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT, env=e)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_prints_one_contract_line():
    from oracle import oracle as O

    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    d = _run(["--impl", "reference", "--workload", "cfg1", "--steps", "2", "--warmup", "1"])
    if "unavailable" in d:
        pytest.skip(d["unavailable"])
    assert d["impl"] == "reference" and d["unit"] == "tokens/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["higher_is_better"] is True and d["dtype"] == "f64" and d["n_gpus"] == 1
    # the same workload the GPU arm reports (BASELINE configs[0] here), its union at full size (3,483
    # on unrounded inputs; 3,484 on the bf16-rounded streams both arms use)
    assert d["config"]["workload"] == "reference_cpu_workload" and d["config"]["global_tokens"] == 256
    assert d["union_size"] == 3484
    assert set(d["phase_seconds"]) == {"select", "fetch", "forward", "backward", "scatter", "adam"}


def test_gpus_flag_launches_that_many_ranks():
    """`bench.py --gpus 2` without a launcher re-executes itself under torch.distributed.run with two ranks (the
    reference arm needs no GPU: both ranks join a gloo rendezvous, rank 0 alone runs and prints)."""
    from oracle import oracle as O

    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    d = _run(["--gpus", "2", "--impl", "reference", "--workload", "cfg1", "--steps", "1", "--warmup", "0"],
             env={"MASTER_ADDR": "127.0.0.1", "GLOO_SOCKET_IFNAME": "lo"})
    assert d["n_gpus"] == 2 and d["ranks_joined"] == 2 and d["config"]["global_tokens"] == 512
    assert d["config"]["parallelism"].startswith("expert-sharded ep2")


def test_mismatched_world_size_fails_loudly():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl", "reference"],
                       capture_output=True, text=True, timeout=120, cwd=ROOT,
                       env=dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0"))
    assert r.returncode != 0 and "WORLD_SIZE=1" in r.stderr


@pytest.mark.gpu
def test_gpu_arm_prints_one_contract_line():
    d = _run(["--steps", "2", "--warmup", "3", "--skip-cpu-baseline"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "roofline", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["config"]["workload"] == "llama7b_meft_layer"
    r = d["roofline"]
    assert r["bound"] == "tensor" and r["unit"] == "TFLOP/s" and 0 < r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["clocks"]["sm_max_mhz"] and isinstance(d["clocks"]["reasons"], list)


def test_reference_arm_reports_unreachable_workloads():
    """BASELINE config 5's M = 4M layer needs 1.1 TB of fp64 HostStore on the host: the reference arm says so
    (one line, exit 0) instead of faking or extrapolating a number."""
    d = _run(["--impl", "reference", "--workload", "cfg5"])
    assert d["impl"] == "reference" and "unavailable" in d and "GB of host RAM" in d["unavailable"]
