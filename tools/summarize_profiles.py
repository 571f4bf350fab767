"""Turns the raw outputs of tools/profile_round.sh (gpurun_out/<R>_*) into the
committed summaries under profiles/: launch-list totals, the ncu full-capture
tables, the traffic JSON and the bench lines.  python tools/summarize_profiles.py [r02]"""
import collections
import csv
import gzip
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
R = sys.argv[1] if len(sys.argv) > 1 else "r02"
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")


def launch_summary():
    rows = list(csv.reader(gzip.open(os.path.join(G, f"{R}_launches_bench.csv.gz"), "rt")))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[hi]
    idx = {h: i for i, h in enumerate(hdr)}
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    for r in rows[hi + 1:]:
        if len(r) < len(hdr) or r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r[idx["Kernel Name"]])
        ms = float(r[idx["Metric Value"]].replace(",", "")) * scale[r[idx["Metric Unit"]]]
        agg[name][0] += 1
        agg[name][1] += ms
        tot += ms
    n = sum(a[0] for a in agg.values())
    out = [f"# ncu launch list of `python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-extras` ({R} code)",
           "# --metrics gpu__time_duration.sum --clock-control none -c 14000 (the list stops at the first 14000 launches); "
           "cold-cache, serialised: compare SHARES. Includes the in-run cuBLAS DGEMM peak measurement",
           "# launches: %d, summed kernel time: %.2f ms" % (n, tot),
           "%-44s %9s %10s %7s" % ("kernel", "launches", "total_ms", "share")]
    for k, (c, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:45]:
        out.append("%-44s %9d %10.3f %6.1f%%" % (k[:44], c, ms, 100 * ms / tot))
    open(os.path.join(P, f"{R}_launch_summary.txt"), "w").write("\n".join(out) + "\n")
    shutil.copy(os.path.join(G, f"{R}_launches_bench.csv.gz"), P)


def ncu_table(rep, title, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}

    def g(r, k):
        try:
            return float(r[idx[k]].replace(",", ""))
        except (KeyError, ValueError):
            return float("nan")

    def mb(r, k):
        v, u = g(r, k), units[idx[k]]
        return v * {"Gbyte": 1e3, "Mbyte": 1.0, "Kbyte": 1e-3, "byte": 1e-6}.get(u, 1.0)

    out.append(title)
    out.append("kernel | grid | block | us | dram_rd_MB | dram_wr_MB | sm_% | dmma_pipe_% | fp64_pipe_% | "
               "lsu_wavefront_% | smem_ld_bank_conflicts | l2_hit_% | warps_% | regs")
    for r in rows[2:]:
        name = r[idx["Kernel Name"]].split("(")[0].replace("void ", "").replace("gmrf::", "")
        t, tu = g(r, "gpu__time_duration.sum"), units[idx["gpu__time_duration.sum"]]
        t *= {"ms": 1e3, "us": 1.0, "ns": 1e-3}.get(tu, 1.0)
        out.append("%s | %s | %s | %.1f | %.1f | %.1f | %.1f | %.1f | %.1f | %.1f | %d | %.1f | %.1f | %d" % (
            name, r[idx["Grid Size"]].strip("()").split(",")[0], r[idx["Block Size"]].strip("()").split(",")[0], t,
            mb(r, "dram__bytes_read.sum"), mb(r, "dram__bytes_write.sum"),
            g(r, "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
            g(r, "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active"),
            g(r, "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
            g(r, "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
            g(r, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"),
            g(r, "lts__t_sector_hit_rate.pct"), g(r, "sm__warps_active.avg.pct_of_peak_sustained_active"),
            g(r, "launch__registers_per_thread")))


def ncu_summary():
    out = []
    big = os.path.join(G, f"{R}_gemm_big.ncu-rep")
    ncu_table(big, "# ncu --set full --clock-control none --import-source on: tools/gemm_big_bench 1 (first shape: the U SYRKs "
              "of five config-5-shape supernodes, r = 8450, K = 1860, ld 10310, row offset 1860; operands 3.8 GB, larger "
              "than L2). k_gemm_tiles = 64x64 tiles / cp.async; k_gemm_wide = 128x128 tiles / cp.async.bulk (TMA) + mbarrier "
              "ring; bit-identical results. Report: profiles/%s_gemm_big.ncu-rep.gz" % R, out)
    out.append("")
    ncu_table(os.path.join(G, f"{R}_full.ncu-rep"),
              "# same options, in situ: python tools/ncu_driver.py (config 4, 1 GN step), "
              "-k regex:k_gemm_tiles|k_panel_|k_extend_add|k_small_front -s 40 -c 20 (mid-tree levels)", out)
    open(os.path.join(P, f"{R}_ncu_summary.txt"), "w").write("\n".join(out) + "\n")
    with open(big, "rb") as f, gzip.open(os.path.join(P, f"{R}_gemm_big.ncu-rep.gz"), "wb") as o:
        shutil.copyfileobj(f, o)


if __name__ == "__main__":
    launch_summary()
    ncu_summary()
    for name in (f"{R}_bench_line.json", f"{R}_bench_reference_line.json", f"{R}_ncu_traffic.json"):
        if os.path.exists(os.path.join(G, name)) and os.path.getsize(os.path.join(G, name)) > 2:
            shutil.copy(os.path.join(G, name), P)
    print(open(os.path.join(P, f"{R}_launch_summary.txt")).read()[:2500])
