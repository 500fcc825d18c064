"""Stall samples per CUDA source line range (warp roles of a warp-specialised kernel).
usage: python tools/role_samples.py <rep> <file> name:lo-hi [name:lo-hi ...]
Lines of other files (inlined helpers) are reported per file."""
import csv, io, subprocess, sys
rep, target = sys.argv[1], sys.argv[2]
ranges = []
for spec in sys.argv[3:]:
    name, rng = spec.split(":")
    lo, hi = map(int, rng.split("-"))
    ranges.append((name, lo, hi))
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
fname, hdr, agg, per_line = None, None, {}, {}
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
    try:
        v = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        ln = int(row[0])
    except ValueError:
        continue
    role = fname
    if fname == target:
        role = next((n for n, lo, hi in ranges if lo <= ln <= hi), target + ":other")
        per_line[ln] = v
    agg[role] = agg.get(role, 0) + v
tot = sum(agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
    print(f"{v:8d} {v / tot * 100:5.1f}%  {k}")
