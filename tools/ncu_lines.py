"""Stall samples per source line, excluding barrier waits, with top reasons.
usage: python tools/ncu_lines.py report.ncu-rep [n] [file-filter]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
filt = sys.argv[3] if len(sys.argv) > 3 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
path = None
lines = []
for r in rows:
    if r and r[0] == "File Path":
        path = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and len(r) > 3 and r[2] == "-":
        cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        vals = {hdr[i][6:]: int(r[i] or 0) for i in cols}
        tot = sum(v for k, v in vals.items() if k != "barrier")
        if tot and filt in path:
            top = sorted(((v, k) for k, v in vals.items() if k != "barrier"), reverse=True)[:3]
            ins = int(r[hdr.index("Instructions Executed")] or 0)
            lines.append((tot, ins, path, r[0], r[1][:70], top))
T = sum(l[0] for l in lines) or 1
print(f"non-barrier stall samples {T}")
for tot, ins, p, ln, src, top in sorted(lines, reverse=True)[:n]:
    print(f"{100*tot/T:5.1f}% {ins:>11d} {p}:{ln:<5} {src:70s} " + " ".join(f"{k}:{100*v/tot:.0f}%" for v, k in top))
