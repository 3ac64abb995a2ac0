"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
        continue
    name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
    v = float(r[hdr.index("Metric Value")].replace(",", ""))
    unit = r[hdr.index("Metric Unit")]
    v = v / 1e6 if unit in ("ns", "nsecond") else v / 1e3 if unit in ("us", "usecond") else v
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':44s} {'launches':>8s} {'total ms':>10s} {'avg us':>9s} {'share':>6s}")
for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:44s} {n:8d} {ms:10.2f} {ms / n * 1e3:9.1f} {100 * ms / tot:5.1f}%")
print(f"{'total (serialised, cold-cache)':44s} {sum(v[0] for v in agg.values()):8d} {tot:10.2f}")
