"""Per-kernel time per step from an ncu launch-list CSV (gpu__time_duration.sum)
of `bench.py --profile --steps 1 --warmup 1` (2 steps captured). Usage:
    python tools/launch_shares.py gpurun_out/launches_X.csv [steps=2]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    nm = r[ki].split("(")[0].replace("void ", "").replace("gqc::<unnamed>::", "")[:70]
    agg[nm][0] += 1
    agg[nm][1] += float(r[vi].replace(",", ""))
tot = sum(v[1] for v in agg.values())
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:16]:
    print(f"{t / 1e6 / steps:9.3f} ms/step {c / steps:6.1f} launches/step {100 * t / tot:5.1f}%  {k}")
