"""Top stall-sampled SASS instructions of one kernel in an ncu report:
python scripts/ncu_hot.py REPORT REGEX [SKIP] [N]"""
import collections
import re
import csv
import subprocess
import sys

rep, rx = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
n = int(sys.argv[4]) if len(sys.argv) > 4 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
# one block per profiled launch ("Kernel Name" line, header, rows); pick the
# skip-th launch whose demangled name matches rx (ncu's own --kernel-name /
# --launch-* filters do not apply to an imported report)
blocks, cur = [], None
for r in csv.reader(out.splitlines()):
    if r and r[0] == "Kernel Name":
        cur = [r]
        blocks.append(cur)
    elif cur is not None:
        cur.append(r)
rows = [b for b in blocks if re.search(rx, b[0][1])][int(skip)]
print(rows[0][1][:100])
hdr = rows[1]
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ci = [hdr.index(c) for c in cols]
isrc, iex = hdr.index("Source"), hdr.index("Instructions Executed")
data, seen, tot = [], set(), collections.Counter()
for r in rows[2:]:
    if len(r) < len(hdr) or r[0] in seen:
        continue
    seen.add(r[0])
    c = collections.Counter()
    for name, i in zip(cols, ci):
        try:
            c[name.replace("stall_", "")] += int(r[i])
        except (ValueError, IndexError):
            pass
    tot.update(c)
    data.append((sum(c.values()), r[0][-5:], r[isrc].strip()[:64], r[iex], c.most_common(2)))
T = sum(tot.values()) or 1
print("samples", T, [(k, round(100 * v / T, 1)) for k, v in tot.most_common(6)])
for d in sorted(data, reverse=True)[:n]:
    print("  %5.1f%% %s %-64s exec=%s %s" % (100 * d[0] / T, d[1], d[2], d[3], d[4]))
