# Power / clock samples while tools/profile_step.py runs (nvidia-smi every 50 ms)
nvidia-smi --query-gpu=power.limit,enforced.power.limit,power.max_limit,clocks.max.sm --format=csv
nvidia-smi --query-gpu=timestamp,power.draw,clocks.sm,clocks.mem,temperature.gpu,clocks_event_reasons.active --format=csv,noheader -lms 50 > gpurun_out/power.csv &
SMI=$!
sleep 1
python tools/profile_step.py 40 epilogue
kill $SMI
python - <<'PY'
import statistics
rows = [l.split(", ") for l in open("gpurun_out/power.csv") if l.strip()]
p = [float(r[1].split()[0]) for r in rows if "W" in r[1]]
c = [float(r[2].split()[0]) for r in rows if "MHz" in r[2]]
busy = [x for x in p if x > 300]
print(f"samples {len(p)}, power under load median {statistics.median(busy) if busy else 0:.0f} W max {max(p):.0f} W, sm clock median {statistics.median(c):.0f} MHz")
PY
