"""Summarise ncu captures into profiles/ (run here, on the CPU box).

usage: python tools/ncu_summary.py <full.ncu-rep> <launches.csv> <out_prefix>
writes <out_prefix>_ncu_full.csv (selected raw metrics per captured kernel),
<out_prefix>_launches.csv (copy) and <out_prefix>_summary.md, and updates
profiles/ncu_traffic_<config>.json (DRAM bytes per launch per kernel, used by bench.py;
the config is the prefix's _cN part, default c2).
"""
import csv
import io
import json
import re
import shutil
import subprocess
import sys
from pathlib import Path

rep, launches, prefix = sys.argv[1], sys.argv[2], sys.argv[3]   # launches: a CSV or "-" (none)
extra = sys.argv[4:]  # optional further launch lists (e.g. the whole bench command), summarised too
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
idx = {w: hdr.index(w) for w in want if w in hdr}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
out_rows = []
traffic = {}
for r in data:
    d = {}
    for w, i in idx.items():
        v, u = r[i], units[i]
        if w.startswith("dram__bytes"):
            v = float(v.replace(",", "")) * scale.get(u, 1)
        d[w] = v
    d["time_unit"] = units[idx["gpu__time_duration.sum"]]
    out_rows.append(d)
    name = d["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "").strip()
    # keep the longest launch per kernel name (the level pass, not the ghat DST of g)
    t = float(str(d["gpu__time_duration.sum"]).replace(",", ""))
    if name not in traffic or t > traffic[name][0]:
        traffic[name] = (t, d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"])
with open(f"{prefix}_ncu_full.csv", "w", newline="") as f:
    w = csv.DictWriter(f, fieldnames=list(out_rows[0].keys()))
    w.writeheader()
    w.writerows(out_rows)
lines = [f"# ncu summary ({Path(prefix).name})"]
ki = vi = None
if launches != "-":
    shutil.copy(launches, f"{prefix}_launches.csv")
    # launch list shares
    lrows = list(csv.reader(open(launches)))
    h = next(i for i, r in enumerate(lrows) if "Kernel Name" in r)
    lh = lrows[h]
    ki, vi = lh.index("Kernel Name"), lh.index("Metric Value")
    agg = {}
    for r in lrows[h + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        agg.setdefault(name, []).append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    lines += ["", "## Launch list (gpu__time_duration.sum, cold-cache, serialised)", "",
              "| kernel | launches | total us | share |", "|---|---|---|---|"]
    for name, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| {name} | {len(v)} | {sum(v)/1e3:.1f} | {sum(v)/tot*100:.1f}% |")
for ex in extra:
    shutil.copy(ex, f"{prefix}_{Path(ex).stem}.csv")
    er = list(csv.reader(open(ex)))
    eh = next(i for i, r in enumerate(er) if "Kernel Name" in r)
    eagg = {}
    for r in er[eh + 1:]:
        if len(r) > vi:
            eagg.setdefault(r[ki].split("(")[0].replace("void ", ""), []).append(float(r[vi].replace(",", "")))
    etot = sum(sum(v) for v in eagg.values())
    lines += ["", f"## Launch list of {Path(ex).name}", "", "| kernel | launches | total us | share |", "|---|---|---|---|"]
    for name, v in sorted(eagg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| {name} | {len(v)} | {sum(v)/1e3:.1f} | {sum(v)/etot*100:.1f}% |")
lines += ["", "## --set full capture (one launch each)", "",
          "| kernel | time | DRAM read | DRAM write | DRAM % | SM % | L1 % | FP64 pipe % | IPC | warps % | regs |",
          "|---|---|---|---|---|---|---|---|---|---|---|"]
for d in out_rows:
    lines.append(f"| {d['Kernel Name'][:48]} | {d['gpu__time_duration.sum']} {d['time_unit']} | "
                 f"{d['dram__bytes_read.sum']/1e9:.3f} GB | {d['dram__bytes_write.sum']/1e9:.3f} GB | "
                 f"{d.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed','')} | "
                 f"{d.get('sm__throughput.avg.pct_of_peak_sustained_elapsed','')} | "
                 f"{d.get('l1tex__throughput.avg.pct_of_peak_sustained_active','')} | "
                 f"{d.get('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active','')} | "
                 f"{d.get('sm__inst_executed.avg.per_cycle_active','')} | "
                 f"{d.get('sm__warps_active.avg.pct_of_peak_sustained_active','')} | "
                 f"{d.get('launch__registers_per_thread','')} |")
Path(f"{prefix}_summary.md").write_text("\n".join(lines) + "\n")
cfg = next((p for p in Path(prefix).name.split("_") if re.fullmatch(r"c[1-5]", p)), "c2")
tj = json.dumps({k: v[1] for k, v in traffic.items()}, indent=1) + "\n"
Path(f"{prefix}_traffic.json").write_text(tj)
if Path("profiles").is_dir():
    Path(f"profiles/ncu_traffic_{cfg}.json").write_text(tj)
print("\n".join(lines))
