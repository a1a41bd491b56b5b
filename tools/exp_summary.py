import json, sys, glob
tag = sys.argv[1]
for f in sorted(glob.glob(f"gpurun_out/exp_{tag}_v*_*.log")):
    L = [l for l in open(f) if l.startswith("{")]
    if not L:
        print(f.split("/")[-1], "FAILED", open(f).read()[-300:].replace("\n", " ")); continue
    d = json.loads(L[-1])
    print(f.split("/")[-1], round(d["value"]), d["engine"]["passes"], d["engine"]["batch_per_gpu"], round(d["roofline"]["frac"], 3),
          d["clocks"]["sm_mhz"])
