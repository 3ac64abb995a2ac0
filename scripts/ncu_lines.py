"""Per-source-line instruction / stall-sample totals of one kernel from an ncu report:
   python scripts/ncu_lines.py REPORT KERNEL_REGEX [TOP]"""
import csv, subprocess, sys
rep, rx = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--kernel-name", f"regex:{rx}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
cur = None
agg = {}
fname = ""
seen_fn = 0
for r in rows:
    if not r:
        continue
    if r[0] == "Kernel Name":
        seen_fn += 1
        if seen_fn > 1:
            break  # first launch only
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if r[0] == "Line No":
        hdr = r
        iE, iS = hdr.index("Instructions Executed"), hdr.index("# Samples")
        continue
    if hdr is None or len(r) < len(hdr) - 2:
        continue
    if r[0] != "":
        cur = (fname, r[0], r[1].strip()[:100])
        agg.setdefault(cur, [0, 0, 0])
        continue
    if cur is None or r[2] in ("...", ""):
        continue
    try:
        e = int(r[iE]); s = int(r[iS])
    except ValueError:
        continue
    a = agg[cur]
    a[0] += e; a[1] += s; a[2] += 1
tot_e = sum(a[0] for a in agg.values()); tot_s = sum(a[1] for a in agg.values())
print(f"total warp-instructions {tot_e}, samples {tot_s}")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{100*a[1]/max(tot_s,1):5.1f}% samp {100*a[0]/max(tot_e,1):5.1f}% inst ({a[2]:4d} sass) {k[0]}:{k[1]}: {k[2]}")
