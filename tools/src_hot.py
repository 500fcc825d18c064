"""Per-CUDA-source-line hot spots from an ncu report (--import-source on, -lineinfo).
usage: python tools/src_hot.py <rep> [n] [kernel-regex] [launch-skip]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"]
if len(sys.argv) > 3:
    cmd += ["-k", "regex:" + sys.argv[3]]
if len(sys.argv) > 4:
    cmd += ["--launch-skip", sys.argv[4], "--launch-count", "1"]
raw = subprocess.run(cmd, capture_output=True, text=True).stdout
out, fname, hdr = [], None, None
for row in csv.reader(io.StringIO(raw)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or row[0] == "" or row[0] == "Function Name":
        continue
    d = dict(zip(hdr[2:], row[2:]))
    def iv(k):
        try:
            return int(d.get(k, "0") or 0)
        except ValueError:
            return 0
    out.append((iv("Warp Stall Sampling (All Samples)"), iv("L1 Wavefronts Shared Excessive"), iv("L1 Wavefronts Shared"),
                iv("Instructions Executed"), f"{fname}:{row[0]}", row[1].strip()[:80]))
tot = sum(o[0] for o in out) or 1
print("samples", tot)
for o in sorted(out, reverse=True)[:n]:
    print(f"{o[0]:6d} {o[0]/tot*100:5.1f}%  smem_wf={o[2]:>9d} excess={o[1]:>9d} inst={o[3]:>10d}  {o[4]:24s} {o[5]}")
