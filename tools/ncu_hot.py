"""Hot CUDA source lines of an ncu report (warp-stall samples by line).
usage: python tools/ncu_hot.py report.ncu-rep [n]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
lines = []
path = None
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "Function Name":
        continue
    try:
        if r[2] != "-":      # a SASS row
            continue
        s = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        ins = int(r[hdr.index("Instructions Executed")])
    except (ValueError, IndexError):
        continue
    lines.append((s, ins, path, r[0], r[1][:100]))
tot = sum(l[0] for l in lines) or 1
print(f"total stall samples {tot}")
for s, ins, p, ln, src in sorted(lines, reverse=True)[:n]:
    print(f"{100*s/tot:5.1f}% {ins:>11d}  {p}:{ln:<5} {src}")


def reasons(rep, line_filter):
    """Stall-reason breakdown for CUDA lines whose number is in line_filter."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    path = None
    for r in rows:
        if r and r[0] == "File Path":
            path = r[1].split("/")[-1]
        elif r and r[0] == "Line No":
            hdr = r
        elif hdr and len(r) > 3 and r[2] == "-" and (path, r[0]) in line_filter:
            cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
            tot = sum(int(r[i]) for i in cols) or 1
            top = sorted(((int(r[i]), hdr[i]) for i in cols), reverse=True)[:5]
            print(path, r[0], r[1][:60], " | ".join(f"{h[6:]} {100*v/tot:.0f}%" for v, h in top))


if __name__ == "__main__" and len(sys.argv) > 3:
    reasons(rep, {tuple(x.split(":")) for x in sys.argv[3].split(",")})
