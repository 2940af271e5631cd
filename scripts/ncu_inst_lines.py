"""Warp-level instructions executed per source line (and per opcode) of an ncu report:
  python scripts/ncu_inst_lines.py report.ncu-rep [n]"""
import collections
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
        i = hdr.index("Instructions Executed")
        try:
            v = float(r[i])
        except ValueError:
            continue
        recs.append((v, cur, int(r[0]), r[1].strip()))
tot = sum(v for v, *_ in recs) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
print(f"total warp instructions {tot:.4g}")
for v, f, ln, src in sorted(recs, reverse=True)[:n]:
    print(f"{v / tot:6.1%} {f}:{ln:<5d} {src[:100]}")
# opcode histogram from the SASS view
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source",
                      "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1] if len(rows) > 1 else []
ops = collections.Counter()
if "Instructions Executed" in h:
    ii, si = h.index("Instructions Executed"), h.index("Source")
    for r in rows[2:]:
        if len(r) == len(h):
            try:
                v = float(r[ii])
            except ValueError:
                continue
            tok = r[si].split()
            op = tok[1] if tok and tok[0].startswith("@") and len(tok) > 1 else (tok[0] if tok else "?")
            ops[op.split(".")[0]] += v
print("opcodes:", ", ".join(f"{k} {v / tot:.1%}" for k, v in ops.most_common(25)))
