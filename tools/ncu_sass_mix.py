#!/usr/bin/env python3
"""Aggregate an ncu '--page source --csv' SASS listing: instruction mix by opcode and stall reasons.
usage: ncu_sass_mix.py <source.csv> [top]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
inst = collections.Counter(); samp = collections.Counter(); stall = collections.Counter()
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    op = r[ix["Source"]].split()[0] if r[ix["Source"]].split() else "?"
    if op.startswith("@"):
        op = r[ix["Source"]].split()[1]
    op = op.split(".")[0]
    inst[op] += float(r[ix["Instructions Executed"]] or 0)
    samp[op] += float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    for h, i in ix.items():
        if h.startswith("stall_") and "Not Issued" not in h:
            stall[h] += float(r[i] or 0)
ti, ts = sum(inst.values()), sum(samp.values())
print(f"instructions {ti:.3e}  samples {ts:.0f}")
for op, v in inst.most_common(top):
    print(f"  {op:10s} inst {v/ti:6.3f}  samples {samp[op]/ts:6.3f}")
st = sum(stall.values())
print("stalls:", ", ".join(f"{k[6:]} {v/st:.2f}" for k, v in stall.most_common(8)))
