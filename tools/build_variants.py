#!/usr/bin/env python3
"""Build library variants (compile-time engine knobs) into paper_1912_02949_b200/lib/variants/.
usage: build_variants.py NAME=DEF1,DEF2 ...   e.g. g0ns3=SCG_NS=3 g1ns3=SCG_GATHER=1,SCG_NS=3"""
import os, subprocess, sys
from concurrent.futures import ThreadPoolExecutor
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1912_02949_b200 as scg
out = os.path.join(scg.LIB_DIR, "variants")
os.makedirs(out, exist_ok=True)
for f in os.listdir(out):
    os.remove(os.path.join(out, f))
jobs = []
for spec in sys.argv[1:]:
    name, defs = spec.split("=", 1)
    jobs.append((name, [d for d in defs.split(",") if d]))
def run(job):
    name, defs = job
    subprocess.check_call(scg.nvcc_cmd(os.path.join(out, name + ".so"), defines=defs), stderr=subprocess.DEVNULL)
    return name
with ThreadPoolExecutor(4) as ex:
    for n in ex.map(run, jobs):
        print("built", n)
