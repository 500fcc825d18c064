"""Top SASS instructions of an ncu source page (stall samples, shared-memory excess).
usage: python tools/sass_hot.py <rep> [kernel-regex] [n]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
args = ["ncu", "-i", rep, "--page", "source", "--csv"]
if len(sys.argv) > 2 and sys.argv[2]:
    args += ["-k", "regex:" + sys.argv[2]]
raw = subprocess.run(args, capture_output=True, text=True).stdout
lines = raw.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
h = rows[0]
ix = {k: h.index(k) for k in h}
data = [r for r in rows[1:] if r and r[0] != "Address" and len(r) == len(h)]
tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
exc = sum(int(r[ix["L1 Wavefronts Shared Excessive"]] or 0) for r in data)
print("total samples", tot, "excess smem wavefronts", exc)
data.sort(key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
for i, r in enumerate(data[:n]):
    print(f'{r[ix["Address"]][-5:]} {int(r[ix["Warp Stall Sampling (All Samples)"]]):6d} '
          f'{int(r[ix["Warp Stall Sampling (All Samples)"]])/tot*100:5.1f}% ex={r[ix["L1 Wavefronts Shared Excessive"]]:>8s} '
          f'{r[ix["Source"]].strip()[:70]}')
print("--- by excess smem wavefronts")
data.sort(key=lambda r: -int(r[ix["L1 Wavefronts Shared Excessive"]] or 0))
for r in data[:12]:
    print(f'{r[ix["Address"]][-5:]} ex={r[ix["L1 Wavefronts Shared Excessive"]]:>8s} wf={r[ix["L1 Wavefronts Shared"]]:>8s} {r[ix["Source"]].strip()[:70]}')
