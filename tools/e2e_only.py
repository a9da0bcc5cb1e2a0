import sys, os, json, time
sys.path.insert(0, os.getcwd())
import bench, paper_1912_02949_b200 as scg, scg_inputs as si
L = si.laplacian("c3"); c = si.CONFIGS["c3"]
for rep in range(2):
    r = bench.run_e2e(scg, si, L, c, 997, 3, 0, {}, 1)
    print(json.dumps(r))
