"""Print the kernel sequence of one cfg2 select step from an ncu launch list."""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
ki, vi = hdr.index('Kernel Name'), hdr.index('Metric Value')
seq = [(r[ki][:44], int(r[vi])) for r in rows[1:]]
which = int(sys.argv[2]) if len(sys.argv) > 2 else 4
idx = [i for i, s in enumerate(seq) if 'k_scan(' in s[0] or 'k_scan<unsigned int>' in s[0]]
i = idx[which]
j = i
while 'k_eval_analytic' not in seq[j][0]:
    j -= 1
for s in seq[j:i + 3]:
    print(f"{s[0]:46s} {s[1] / 1000:8.2f} us")
print(f"prep total {sum(s[1] for s in seq[j:i]) / 1000:.2f} us")
