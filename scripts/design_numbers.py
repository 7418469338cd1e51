"""Markdown tables for DESIGN.md section 5 from a bench.py JSON line."""
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
cpu = d["cpu_baseline"]
r = d["roofline"]
e = d["e2e"]
st = d["stages_ms_per_step"]
print("  | Measurement | B200 | CPU port (%d cores, %s) |" % (cpu["cores"], cpu.get("cpu_model", "?")))
print("  |---|---|---|")
print("  | C5 c128 WB-arSVD (headline) | **%s updates/s** (%.3f s/step; round 1: 3,933 incl. channels; start of this session: 7,885) | %.0f updates/s |"
      % (f"{d['value']:,.0f}", d["ms_per_step"] / 1e3, cpu["value"]))
print("  | C5 c128 full inversion | %s updates/s | — |" % f"{d['full_inverse']['value']:,.0f}")
print("  | C5 c128 e2e (pinned host H, %d trials × 100 steps, H2D overlapped) | %s updates/s (PCIe: %.0f GB H2D per step) | — |"
      % (e["trials_per_gpu"], f"{e['value']:,.0f}", e["h2d_bytes_per_step"] / 1e9))
fp = r.get("four_product_equivalent")
print("  | dominant kernel | %s: %.1f %s executed = **%.2f of FP64 peak**%s, DRAM %.2f GB/launch vs %.2f GB algorithmic | — |"
      % (r["kernel"], r["achieved"], r["unit"], r["frac"],
         (" (%.1f TFLOP/s = %.2f of it in SURVEY 8(d)'s four-product flops)" % (fp["achieved"], fp["frac"])) if fp else "",
         (r.get("traffic") or 0) / 1e9, r["algorithmic"]["bytes_per_launch"] / 1e9))
print()

print("  | Config | WB updates/s | Full updates/s | Dominant kernel (frac) | CPU |")
print("  |---|---|---|---|---|")
def fmt(v):
    return f"{v / 1e6:.2f} M" if v >= 1e6 else f"{v / 1e3:.1f} K"
c4 = {}
for k, v in d["configs"].items():
    wb = [x for x in v if x.startswith("wb_")]
    w = v[wb[0]] if wb else None
    f = v.get("conventional")
    rr = (w or f).get("roofline") or {}
    cpu_v = v.get("cpu_baseline", {}).get("value")
    if k.startswith("C4"):
        c4[k] = (w["updates_per_s"], f["updates_per_s"] if f else None, rr, cpu_v)
        continue
    print("  | %s | %s | %s | %s (%.2f) | %s |" % (k.replace("_", " "), fmt(w["updates_per_s"]) if w else "—",
          fmt(f["updates_per_s"]) if f else "—", rr.get("kernel"), rr.get("frac", 0),
          fmt(cpu_v) if cpu_v else "—"))
if c4:
    caps = {}
    for k, (w, f, rr, cv) in c4.items():
        cap = k.split("_")[1]
        caps.setdefault(cap, []).append(w)
    line = ", ".join(f"{c} {fmt(sum(v) / len(v))}" for c, v in caps.items())
    ff = [f for (_, f, _, _) in c4.values() if f][0]
    cv = [c for (_, _, _, c) in c4.values() if c][0]
    rr = list(c4.values())[0][2]
    print("  | C4 c64, 12 cap × tol runs (mean over tol) | %s | %s | %s (%.2f) | %s |"
          % (line, fmt(ff), rr.get("kernel"), rr.get("frac", 0), fmt(cv)))
leo = d.get("leo_campaign")
if leo:
    print("  | LEO default campaign (`run_campaign`) | %s | — | — | %s |" % (fmt(leo["value"]), fmt(leo["cpu_baseline"]["value"])))
print()
print("* Stage split at C5 c128 per step (ms, unpipelined pass): " + ", ".join(f"{k} {v:.0f}" for k, v in st.items() if v >= 0.5) + ".")
