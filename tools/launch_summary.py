#!/usr/bin/env python3
"""Summarize an ncu launch list (gpu__time_duration.sum per launch): per-kernel count, mean, share.
usage: launch_summary.py launches.csv [skip_first_n_launches]"""
import csv, sys, collections
path = sys.argv[1]
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rows = [l for l in open(path) if l.startswith('"')]
rd = list(csv.DictReader(rows))
tot = collections.defaultdict(float); cnt = collections.Counter()
for r in rd[skip:]:
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0].replace("void ", "")
    us = float(r["Metric Value"]) / (1000.0 if r["Metric Unit"] == "ns" else 1.0)
    tot[name] += us; cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':32s} {'launches':>8s} {'mean_us':>10s} {'total_us':>12s} {'share':>7s}")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k:32s} {cnt[k]:8d} {tot[k]/cnt[k]:10.1f} {tot[k]:12.1f} {tot[k]/T:7.3f}")
print(f"{'TOTAL':32s} {sum(cnt.values()):8d} {'':10s} {T:12.1f}")
