"""Dev helper: per-source-line instruction and stall-sample shares from
`ncu -i rep --page source --csv --print-source cuda,sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
fname, out = "?", []
for r in rows:
    if r and r[0] == "File Name":
        fname = r[1].split("/")[-1]
    elif r and r[0].isdigit() and len(r) > 8:
        try:
            out.append((fname, int(r[0]), r[1][:80], float(r[7] or 0), float(r[4] or 0)))
        except ValueError:
            pass
ti = sum(o[3] for o in out) or 1
ts = sum(o[4] for o in out) or 1
for f, ln, src, ins, st in sorted(out, key=lambda o: -o[4])[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{f:18s}:{ln:<5d} instr {100 * ins / ti:5.1f}%  stall {100 * st / ts:5.1f}%  {src}")
print(f"total instructions {ti:.3e}")
