"""Top source lines by warp-stall samples from an ncu report (needs -lineinfo)."""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source",
                      "sass,cuda"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur, hdr, recs = None, None, []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
    elif len(r) > 2 and r[0] == "Line No":
        hdr = r
    elif hdr and len(r) == len(hdr) and r[0].isdigit():
        i = hdr.index("Warp Stall Sampling (All Samples)")
        try:
            v = float(r[i])
        except ValueError:
            continue
        recs.append((v, cur, int(r[0]), r[1].strip()))
tot = sum(v for v, *_ in recs) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for v, f, ln, src in sorted(recs, reverse=True)[:n]:
    print(f"{v / tot:6.1%} {f}:{ln:<5d} {src[:100]}")
