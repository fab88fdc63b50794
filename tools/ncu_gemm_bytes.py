"""Per-launch time and DRAM bytes of the GEMM kernels in an ncu --metrics CSV (developer helper)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi or "gemm" not in r[ki]:
        continue
    d.setdefault(r[ii], {"k": r[ki].split("(")[0].split("::")[-1]})[r[mi]] = float(r[vi].replace(",", ""))
for k, v in d.items():
    print(f"{k:>4} {v['k']:28s} ms={v['gpu__time_duration.sum'] / 1e6:.3f} "
          f"rd={v['dram__bytes_read.sum'] / 1e9:.2f}GB wr={v['dram__bytes_write.sum'] / 1e9:.2f}GB")
