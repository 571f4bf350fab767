"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Metric Name" in r)
h = rows[hdr]
ki, mi, ui, vi = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
tot, cnt = defaultdict(float), defaultdict(int)
scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}
for r in rows[hdr + 1:]:
    if len(r) < len(h) or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0]
    tot[name] += float(r[vi].replace(",", "")) * scale[r[ui]]
    cnt[name] += 1
all_ms = sum(tot.values())
print("# launches: %d, summed kernel time: %.2f ms" % (sum(cnt.values()), all_ms))
print("%-44s %8s %10s %7s" % ("kernel", "launches", "total_ms", "share"))
for k in sorted(tot, key=lambda k: -tot[k]):
    print("%-44s %8d %10.3f %6.1f%%" % (k[:44], cnt[k], tot[k], 100 * tot[k] / all_ms))
