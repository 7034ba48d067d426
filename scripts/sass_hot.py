"""Dev helper: hottest SASS instructions of an ncu report (source page)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
hdr = rows[0]
ci = hdr.index("Instructions Executed")
cs = hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[1:]:
    if len(r) != len(hdr):
        continue
    try:
        data.append((int(r[ci] or 0), int(r[cs] or 0), r[0], r[1]))
    except ValueError:
        pass
tot_i = sum(d[0] for d in data)
tot_s = sum(d[1] for d in data)
print(f"instructions {tot_i}, stall samples {tot_s}")
mode = sys.argv[3] if len(sys.argv) > 3 else "samples"
key = (lambda d: d[1]) if mode == "samples" else (lambda d: d[0])
for d in sorted(data, key=key, reverse=True)[:top]:
    print(f"{d[0]:>11} {100*d[0]/max(tot_i,1):5.1f}%  {d[1]:>7} {100*d[1]/max(tot_s,1):5.1f}%  {d[2]}  {d[3]}")
