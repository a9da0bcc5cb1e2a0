"""Bucket PC-sampling stall samples of one ncu report by SASS region: python tools/ncu_regions.py REP [bucket_hex]"""
import csv, subprocess, sys, collections, io
rep = sys.argv[1]; bk = int(sys.argv[2], 16) if len(sys.argv) > 2 else 0x400
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]; iS = h.index("Warp Stall Sampling (All Samples)"); iE = h.index("Instructions Executed")
seen = set(); ins = []
for r in rows[2:]:
    if len(r) < 5 or not r[0].startswith("0x") or r[0] in seen: continue
    seen.add(r[0]); ins.append((int(r[0], 16), float(r[iS] or 0), float(r[iE] or 0), r[1].strip()))
base = ins[0][0]; tot = sum(s for _, s, _, _ in ins)
b = collections.OrderedDict()
for a, s, e, t in ins:
    k = (a - base) // bk
    b.setdefault(k, [0, 0, ""]); b[k][0] += s; b[k][1] += e
    if s > 0.02 * tot and not b[k][2]: b[k][2] = t[:60]
print("total samples", tot)
for k, (s, e, t) in b.items():
    if s > 0.01 * tot: print(f"{k * bk:6x} {100 * s / tot:5.1f}% inst={int(e):9d} {t}")
