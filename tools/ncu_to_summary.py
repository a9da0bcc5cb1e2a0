#!/usr/bin/env python3
"""Record one kernel's ncu --set full capture in profiles/ncu_full_summary.json (read by bench.py for
the roofline "traffic" figure) and write its text summary next to it.

usage: python tools/ncu_to_summary.py <report.ncu-rep> <kernel class name> <workload> <round> <source note>
   e.g. python tools/ncu_to_summary.py gpurun_out/r02d/prof_k_lanczos_a.ncu-rep lanczos_a_spmv_dot c3 r02 "..."
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep, cls, workload, rnd, note = sys.argv[1:6]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
launches = [dict(zip(hdr, r)) for r in rows[2:]]
if not launches:
    raise SystemExit("no launches in " + rep)


def num(d, k):
    v = d.get(k, "")
    return float(v.replace(",", "")) if v not in ("", "n/a") else float("nan")


# ncu reports dram bytes in the unit of the header row (Mbyte / Gbyte / byte): normalise to bytes
units = dict(zip(hdr, rows[1]))
scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def nbytes(d, k):
    return num(d, k) * scale.get(units.get(k, "byte"), 1.0)


rd = sum(nbytes(d, "dram__bytes_read.sum") for d in launches) / len(launches)
wr = sum(nbytes(d, "dram__bytes_write.sum") for d in launches) / len(launches)
tu = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(units.get("gpu__time_duration.sum", "usecond"), 1.0)
dur = sum(num(d, "gpu__time_duration.sum") for d in launches) / len(launches) * tu
path = os.path.join(ROOT, "profiles", "ncu_full_summary.json" if workload == "c3" else f"ncu_full_summary_{workload}.json")
try:
    js = json.load(open(path))
except Exception:
    js = {}
if js.get("workload") != workload or js.get("round") != rnd:
    js = {"workload": workload, "round": rnd, "kernels": {}}
js["source"] = note
js["kernels"][cls] = {"ncu_name": launches[0]["Kernel Name"].split("(")[0], "launches_captured": len(launches),
                      "dram_bytes": round(rd + wr), "dram_read": round(rd), "dram_write": round(wr),
                      "duration_us": round(dur, 2), "registers": int(num(launches[0], "launch__registers_per_thread")),
                      "inst_executed": int(num(launches[0], "smsp__inst_executed.sum"))}
with open(path, "w") as f:
    json.dump(js, f, indent=1)
    f.write("\n")
print(json.dumps(js["kernels"][cls], indent=1))
