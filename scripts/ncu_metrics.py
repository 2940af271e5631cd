"""Print selected raw metrics per kernel launch from an ncu report."""
import csv
import io
import subprocess
import sys

M = sys.argv[2].split(",")
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv", "--metrics", ",".join(M)],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
for r in rows[2:]:
    print(r[hdr.index("Kernel Name")][:60], r[hdr.index("Grid Size")])
    for m in M:
        if m in hdr:
            print(f"    {m:90s} {r[hdr.index(m)]}")
