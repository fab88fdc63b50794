"""Per-launch (ms, DRAM GB read, GHz[, tensor-active %, active tensor Gcycles/s]) of the last step's six FFN GEMMs
from tools/ab_*.sh ncu csv files."""
import collections
import csv
import sys

for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    mi, vi, ii, ui = h.index("Metric Name"), h.index("Metric Value"), h.index("ID"), h.index("Metric Unit")
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3,
             "Gbyte": 1.0, "hz": 1e-9, "Khz": 1e-6, "Mhz": 1e-3, "Ghz": 1.0, "cycle/second": 1e-9,
             "cycle/nsecond": 1.0, "cycle/usecond": 1e-3}
    d = collections.defaultdict(dict)
    for r in rows[hi + 1:]:
        d[int(r[ii])][r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    ids = sorted(d)[-6:]
    tot = sum(d[i]["gpu__time_duration.sum"] for i in ids)
    tensor = "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
    print(path.split("/")[-1], f"sum {tot:.3f} ms",
          [(round(d[i]["gpu__time_duration.sum"], 3), round(d[i]["dram__bytes_read.sum"], 1),
            round(d[i]["sm__cycles_elapsed.avg.per_second"], 2))
           + ((round(d[i][tensor], 1), round(d[i][tensor] * d[i]["sm__cycles_elapsed.avg.per_second"] / 100, 3))
              if tensor in d[i] else ()) for i in ids])
