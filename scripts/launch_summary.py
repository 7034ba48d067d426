"""Dev helper: per-kernel totals from an ncu --csv launch list."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
tot, cnt = {}, {}
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            k = d["Kernel Name"][:100]
            v = float(d["Metric Value"]) * (1e-3 if d.get("Metric Unit") == "nsecond" else 1.0)
            tot[k] = tot.get(k, 0.0) + v
            cnt[k] = cnt.get(k, 0) + 1
all_us = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v:10.1f} us {100 * v / all_us:5.1f}% x{cnt[k]:<4d} {k}")
print(f"{all_us:10.1f} us total, {sum(cnt.values())} launches")
