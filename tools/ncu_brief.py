"""Key metrics + opcode histogram of a one-kernel ncu report: python tools/ncu_brief.py <rep> [kernel-regex]"""
import collections, csv, io, re, subprocess, sys

rep = sys.argv[1]
kargs = ["-k", "regex:" + sys.argv[2]] if len(sys.argv) > 2 else []
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"] + kargs, capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, units, v = r[0], r[1], r[2]
pat = (r"gpu__time_duration.sum|dram__bytes_(read|write).sum$|l1tex__data_pipe_lsu_wavefronts_mem_shared.sum$|"
       r"l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum$|pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active|"
       r"l1tex__throughput.avg.pct_of_peak_sustained_active|sm__warps_active.avg.pct|smsp__inst_executed.sum$|"
       r"launch__registers_per_thread$|pcsamp_sample_count")
for i, n in enumerate(h):
    if re.search(pat, n):
        print(f"{n:70s} {units[i]:8s} {v[i]}")
st = {n.split("stalled_")[1]: float(v[i]) for i, n in enumerate(h)
      if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued") and v[i]}
tot = sum(st.values()) or 1
print("stalls:", ", ".join(f"{k} {x / tot * 100:.0f}%" for k, x in sorted(st.items(), key=lambda t: -t[1]) if x / tot > 0.02))
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] + kargs,
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
start = next(i for i, x in enumerate(rows) if x and x[0] == "Address")
ix = {k: i for i, k in enumerate(rows[start])}
c = collections.Counter()
for x in rows[start + 1:]:
    if len(x) <= ix["Instructions Executed"] or x[0] == "Address":
        continue
    n = int(x[ix["Instructions Executed"]] or 0)
    op = x[ix["Source"]].strip().split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    c[o.split(".")[0]] += n
t = sum(c.values()) or 1
print("ops:", ", ".join(f"{o} {n / t * 100:.1f}%" for o, n in c.most_common(14)), f"(total {t})")
