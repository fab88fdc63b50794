"""Developer probe (CPU, reference only): how the unmodified reference's sparse_ffn_pa / sparse_backward cost grows
with the number of token rows at the cfg2 table shapes (|S| = 65,536), to separate the per-call fixed cost (the
serial 2 GB transposes and d x |S| outputs of sparse_backward) from the per-row cost.
  python tools/ref_cost_curve.py [rows ...]   -> one JSON line per row count"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    rows_list = [int(x) for x in sys.argv[1:]] or [1, 16, 64, 256]
    bench.CFG.update(bench.WORKLOADS["cfg2"])
    from oracle import oracle as O

    O.ref().ref_set_threads(os.cpu_count())
    st, h, g = bench.reference_inputs()
    t0 = time.perf_counter()
    r = st.step_phases(0, h, g, 4, 128, 1e-4, [(0, n) for n in rows_list])
    print(json.dumps({"cores": os.cpu_count(), "select": r["select"], "fetch": r["fetch"], "scatter": r["scatter"],
                      "adam": r["adam"], "wall": time.perf_counter() - t0}), flush=True)
    for n, f, b in zip(rows_list, r["forward"], r["backward"]):
        print(json.dumps({"rows": n, "forward_s": f, "backward_s": b}), flush=True)


if __name__ == "__main__":
    main()
