"""Summarise ncu output into text for profiles/.

    python scripts/ncu_summary.py launches gpurun_out/launches.csv
    python scripts/ncu_summary.py report gpurun_out/prof_x.ncu-rep
"""

import collections
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Ipc Active", "Issue Slots Busy",
        "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Achieved Active Warps Per SM", "Executed Instructions", "Block Size", "Grid Size",
        "Warp Cycles Per Issued Instruction", "Static Shared Memory Per Block",
        "Dynamic Shared Memory Per Block", "FP64", "Fp64"]


def launches(path):
    """Per-kernel launch count, time and DRAM bytes from a --metrics launch list
    (one CSV row per (launch, metric))."""
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    mi = h.index("Metric Name")
    tscale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    bscale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
    agg = collections.OrderedDict()   # name -> [launches, ms, DRAM MB]
    for r in data:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        v = float(r[vi].replace(",", ""))
        e = agg.setdefault(name, [0, 0.0, 0.0])
        if r[mi] == "gpu__time_duration.sum":
            e[0] += 1
            e[1] += v * tscale.get(r[ui], 1e-6)
        elif r[mi].startswith("dram__bytes"):
            e[2] += v * bscale.get(r[ui], 1e-6)
    tot = sum(v[1] for k, v in agg.items() if "cutlass" not in k)
    print(f"{'launches':>8} {'total ms':>10} {'ms/launch':>10} {'MB/launch':>10} {'share':>6}  kernel "
          "(cold-cache, serialised; cuBLAS peak-measurement GEMMs excluded from share)")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        if v[0] == 0:
            continue
        share = "" if "cutlass" in k else f"{100 * v[1] / tot:5.1f}%"
        print(f"{v[0]:8d} {v[1]:10.3f} {v[1] / v[0]:10.4f} {v[2] / v[0]:10.1f} {share:>6}  {k[:90]}")


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    kname = None
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Kernel Name") != kname:
            kname = d.get("Kernel Name")
            print(f"== {kname}")
        n = d.get("Metric Name", "")
        if any(k in n for k in KEYS):
            print(f"  {d.get('Section Name', '')[:28]:28s} {n[:48]:48s} {d.get('Metric Value', '')} "
                  f"{d.get('Metric Unit', '')}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) >= 3:
        hh, units, vals = rr[0], rr[1], rr[2]
        for want in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                     "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                     "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
                     "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
                     "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
                     "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active"):
            for i, name in enumerate(hh):
                if name == want:
                    print(f"  raw {name:60s} {vals[i]} {units[i]}")


def traffic(path, out=None):
    """Per-kernel launches, mean duration and mean DRAM bytes per launch from an
    ncu --csv log with gpu__time_duration.sum, dram__bytes_read.sum and
    dram__bytes_write.sum; optionally written as JSON (read by bench.py)."""
    import json
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, ii = h.index("Kernel Name"), h.index("ID")
    gi = h.index("Grid Size")
    mi, vi, ui = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    per = {}
    for r in data:
        if len(r) <= vi:
            continue
        # one template instantiation serves several products: key by grid size too
        key = (r[ii], r[ki].split("(")[0] + " grid" + r[gi].replace(" ", ""))
        d = per.setdefault(key, {})
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        if r[mi] == "gpu__time_duration.sum":
            v *= {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0,
                  "msecond": 1.0}.get(unit, 1e-6)
        else:
            v *= {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)
        d[r[mi]] = v
    agg = {}
    for (_, name), d in per.items():
        a = agg.setdefault(name, {"launches": 0, "ms": 0.0, "dram_bytes": 0.0})
        a["launches"] += 1
        a["ms"] += d.get("gpu__time_duration.sum", 0.0)
        a["dram_bytes"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    res = {k: {"launches": v["launches"], "ms_per_launch": v["ms"] / v["launches"],
               "dram_bytes_per_launch": v["dram_bytes"] / v["launches"]} for k, v in agg.items()}
    for k, v in sorted(res.items(), key=lambda x: -x[1]["ms_per_launch"] * x[1]["launches"]):
        print(f"{v['launches']:6d} {v['ms_per_launch']:9.4f} ms {v['dram_bytes_per_launch'] / 1e6:10.1f} MB  {k[:80]}")
    if out:
        with open(out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    fn = {"launches": launches, "report": report, "traffic": traffic}[sys.argv[1]]
    fn(*sys.argv[2:])
