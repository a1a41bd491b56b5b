"""Summaries of a gpu_round.sh run for profiles/ (tracked):
   python tools/make_profiles.py TAG OUTPREFIX
writes OUTPREFIX_launches_config4.txt, OUTPREFIX_pass_kernels_ncu.txt, OUTPREFIX_bench_line.json,
OUTPREFIX_bench_reference_line.json and profiles/pass_traffic_config4.json (read by bench.py)."""
import collections, csv, io, json, subprocess, sys
from contextlib import redirect_stdout
from pathlib import Path

tag, out = sys.argv[1], sys.argv[2]
fill_csv = sys.argv[3] if len(sys.argv) > 3 else None
G = Path("gpurun_out")
# launch list
rows = list(csv.reader(open(G / f"launches_{tag}.csv")))
hdr, agg = None, collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or len(r) < len(hdr) or r[hdr["Metric Name"]] != "gpu__time_duration.sum":
        continue
    k = r[hdr["Kernel Name"]][:48]
    v = float(r[hdr["Metric Value"]].replace(",", "")) * {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
                                                          "second": 1e3}.get(r[hdr["Metric Unit"]], 1.0)
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(a[1] for a in agg.values())
with open(f"{out}_launches_config4.txt", "w") as f:
    f.write("ncu --metrics gpu__time_duration.sum --clock-control none -c 600: python bench.py --steps 2 --warmup 3 "
            "--no-cpu\nconfig 4 (28 q, c64), batch 48, shared-trunk schedule; per-launch device time (serialised, "
            "cold cache: compare SHARES)\n")
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        f.write(f"{k:48s} launches={a[0]:4d} total_ms={a[1]:10.2f} share={100 * a[1] / tot:5.1f}% "
                f"avg_ms={a[1] / a[0]:8.3f}\n")
    passes = sum(a[1] for k, a in agg.items() if k.startswith("ptsbe_pass"))
    f.write(f"pass kernels share of all device time: {100 * passes / tot:.1f}%\n")
# ncu full table of every pass kernel of one step
buf = io.StringIO()
with redirect_stdout(buf):
    sys.argv = ["ncu_table", str(G / f"pass_raw_{tag}.csv")]
    exec(open("tools/ncu_table.py").read())
with open(f"{out}_pass_kernels_ncu.txt", "w") as f:
    f.write("ncu --set full --clock-control none -k regex:ptsbe_pass -s 36 -c 12: the 12 pass launches of one bench "
            "step (config 4)\n(time column in ncu units, serialised replay: compare shares; GB = dram read+write)\n")
    f.write(buf.getvalue())
# traffic per pass launch (dram bytes) for bench.py
rows = list(csv.reader(open(G / f"pass_raw_{tag}.csv")))
h = {k: i for i, k in enumerate(rows[0])}
units = rows[1]
def val(r, k):
    return float(r[h[k]].replace(",", "")) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "Tbyte": 1e12}.get(
        units[h[k]], 1)
by = [val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum") for r in rows[2:]]
names = [r[h["Kernel Name"]] for r in rows[2:]]
# ncu occasionally reports -nan DRAM counters for a long kernel under --set full: fill those
# from a targeted --metrics capture (optional 3rd argument: its --csv log)
if fill_csv:
    fill = collections.defaultdict(float)
    hh = None
    for r in csv.reader(open(fill_csv)):
        if r and r[0] == "ID":
            hh = {k: i for i, k in enumerate(r)}
            continue
        if hh and len(r) > 10 and r[hh["Metric Name"]].startswith("dram__bytes"):
            fill[r[hh["Kernel Name"]]] += float(r[hh["Metric Value"]].replace(",", "")) * (
                1 if r[hh["Metric Unit"]] == "byte" else {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[r[hh["Metric Unit"]]])
    by = [fill[nm] if (b != b and nm in fill) else b for b, nm in zip(by, names)]
json.dump({"per_launch_dram_bytes": sum(by) / len(by), "launches": len(by), "per_pass_dram_bytes": by,
           "config": 4, "batch_per_gpu": 48, "dtype": "c64",
           "source": f"ncu --set full of the {len(by)} pass launches of one bench step (gpurun tag {tag})"
                     + (f"; -nan counters refilled from a targeted --metrics capture" if fill_csv else "")},
          open("profiles/pass_traffic_config4.json", "w"), indent=1)
for name, src in (("bench_line", f"bench_{tag}.log"), ("bench_reference_line", f"bench_ref_{tag}.log")):
    for line in open(G / src):
        if line.startswith("{"):
            open(f"{out}_{name}.json", "w").write(line)
print("ok", tot)
