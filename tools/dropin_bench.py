"""The MEFT layer step through the reference's public C++ API (meft_ffn -> sparse_backward -> scatter_grads ->
sparse_adam_update, host tables in and out) with the reference library vs the drop-in library
(tests/dropin/layer_bench.cpp built both ways), at BASELINE config 1 and at the LLaMA width with T = 64 (a sparse
union). Prints one JSON line per (config, library) with the median step and its phases.
  python tools/dropin_bench.py [out.jsonl]"""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXES = {"reference": os.path.join(ROOT, "oracle", "_ref", "tests", "layer_bench"),
        "dropin": os.path.join(ROOT, "build", "dropin_tests", "layer_bench")}
CONFIGS = [("cfg1", (512, 4096, 64, 32, 4, 256), 5), ("llama_width_T64", (4096, 65536, 256, 128, 4, 64), 2)]


def main():
    out = open(sys.argv[1], "w") if len(sys.argv) > 1 else None
    for name, shape, steps in CONFIGS:
        for lib, exe in EXES.items():
            r = subprocess.run([exe] + [str(x) for x in shape] + [str(steps)], capture_output=True, text=True,
                               timeout=3600)
            if r.returncode != 0:
                line = {"config": name, "library": lib, "error": r.stderr[-500:]}
            else:
                rows = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
                med = statistics.median(x["step_s"] for x in rows)
                best = min(rows, key=lambda x: abs(x["step_s"] - med))
                line = {"config": name, "library": lib, "shape": dict(zip("d M N K kk T".split(), shape)),
                        "cores": os.cpu_count(), "steps": len(rows), "median_step_s": med,
                        "tokens_per_s": shape[5] / med, "phases_s": {k: best[k] for k in best if k.endswith("_s")},
                        "union": best["union"]}
            print(json.dumps(line), flush=True)
            if out:
                out.write(json.dumps(line) + "\n")


if __name__ == "__main__":
    main()
