"""DRAM traffic per launch of the GEMM tile kernel from an ncu metrics CSV.

  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      -k regex:k_gemm_ --csv --log-file gemm_traffic.csv \
      python tools/ncu_driver.py 999 1000
  python tools/ncu_traffic.py gemm_traffic.csv > profiles/r02_ncu_traffic.json

Keyed by the bench's kernel class (factor.gemm_dmma: every k_gemm_tiles /
k_gemm_next / k_gemm_wide launch of one config-4 posterior with one GN step —
three factorizations + the selected inversion, whose GEMM launches share the
kernels)."""
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Metric Name" in r)
h = rows[hdr]
idx = {k: h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value")}
per = {}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3}
for r in rows[hdr + 1:]:
    if len(r) < len(h) or "k_gemm_" not in r[idx["Kernel Name"]]:
        continue
    v = float(r[idx["Metric Value"]].replace(",", "")) * scale.get(r[idx["Metric Unit"]], 1)
    per.setdefault(r[idx["ID"]], {})[r[idx["Metric Name"]]] = v
n = len(per)
dram = sum(p.get("dram__bytes_read.sum", 0) + p.get("dram__bytes_write.sum", 0) for p in per.values())
t = sum(p.get("gpu__time_duration.sum", 0) for p in per.values())
print(json.dumps({"factor.gemm_dmma": {
    "dram_bytes_per_launch": dram / max(n, 1), "launches_sampled": n,
    "dram_gbs_while_running": dram / max(t, 1e-12) / 1e9,
    "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (cold cache, serialised) over "
              "every k_gemm_* launch of tools/ncu_driver.py 999 1000", "workload": "c4"}}, indent=1))
