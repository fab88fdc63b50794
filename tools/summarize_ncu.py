"""Summarise ncu outputs into the text files committed under profiles/.

  python tools/summarize_ncu.py launches <launches.csv>     per-kernel share of device time (launch list)
  python tools/summarize_ncu.py full <report.ncu-rep>       key metrics of a --set full capture
  python tools/summarize_ncu.py traffic <report.ncu-rep> <out.json>
                                                            mean per-launch DRAM bytes of the captured kernels
                                                            (bench.py reports it as roofline.traffic)
"""
import collections
import csv
import io
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        if len(r) <= vi:
            continue
        ms = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        name = r[ki].split("(")[0].replace("void ", "").replace("meft_dev::<unnamed>::", "")
        agg[name][0] += 1
        agg[name][1] += ms
    tot = sum(v[1] for v in agg.values())
    print(f"{'total ms':>10} {'share':>6} {'launches':>8} {'ms/launch':>10}  kernel")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{v[1]:10.3f} {100 * v[1] / tot:5.1f}% {v[0]:8d} {v[1] / v[0]:10.4f}  {k}")


KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__inst_executed.sum"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        print("kernel:", v[h.index("Kernel Name")][:120])
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"  {k} = {v[i]} {u[i]}")


def traffic(path, out_json):
    import json
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    per = []
    for v in rows[2:]:
        b = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = h.index(k)
            b += float(v[i].replace(",", "")) * unit[u[i]]
        per.append({"kernel": v[h.index("Kernel Name")].split("(")[0].split("::")[-1], "dram_bytes": b,
                    "ms": float(v[h.index("gpu__time_duration.sum")].replace(",", "")) *
                    {"ms": 1, "msecond": 1, "us": 1e-3, "usecond": 1e-3}[u[h.index("gpu__time_duration.sum")]]})
    res = {"source": path.split("/")[-1], "launches": per,
           "mean_dram_bytes_per_launch": sum(p["dram_bytes"] for p in per) / len(per)}
    json.dump(res, open(out_json, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    {"launches": launches, "full": full, "traffic": traffic}[sys.argv[1]](*sys.argv[2:])
