"""Summaries of a tools/gpu_prof_r2.sh run for profiles/ (tracked):

   python tools/make_profiles_r2.py TAG OUTPREFIX [BATCH_c128 BATCH_c64]

For each dtype (c128, c64): OUTPREFIX_launches_config4_<dtype>.txt (kernel shares of
the ncu launch list of a 2-step bench run), OUTPREFIX_pass_dram_config4_<dtype>.csv (the
raw per-pass-launch DRAM/time capture, kept as provenance) and
profiles/pass_traffic_config4_<dtype>.json (DRAM bytes per pass launch, read by bench.py
for roofline.traffic when config / batch / dtype / pass count match)."""
import collections
import csv
import json
import shutil
import sys
from pathlib import Path

tag, out = sys.argv[1], sys.argv[2]
batch = {"c128": int(sys.argv[3]) if len(sys.argv) > 3 else 24, "c64": int(sys.argv[4]) if len(sys.argv) > 4 else 48}
G = Path("gpurun_out")
UNIT = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3}
BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def rows_of(path):
    hdr = None
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = {h: i for i, h in enumerate(r)}
            continue
        if hdr is not None and len(r) >= len(hdr):
            yield hdr, r


for d in ("c128", "c64"):
    lf = G / f"launches_{d}_{tag}.csv"
    if lf.exists():
        agg = collections.OrderedDict()
        for h, r in rows_of(lf):
            if r[h["Metric Name"]] != "gpu__time_duration.sum":
                continue
            k = r[h["Kernel Name"]][:48]
            v = float(r[h["Metric Value"]].replace(",", "")) * UNIT.get(r[h["Metric Unit"]], 1.0)
            a = agg.setdefault(k, [0, 0.0])
            a[0] += 1
            a[1] += v
        tot = sum(a[1] for a in agg.values())
        with open(f"{out}_launches_config4_{d}.txt", "w") as f:
            f.write(f"ncu --metrics gpu__time_duration.sum --clock-control none -c 1000: python bench.py --steps 2 "
                    f"--warmup 3 --no-cpu --dtype {d} --secondary none\nconfig 4 (28 q, {d}), batch {batch[d]}, "
                    "shared-trunk schedule, Philox shots; per-launch device time (serialised, cold cache: compare "
                    "SHARES)\n")
            for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
                f.write(f"{k:48s} launches={a[0]:4d} total_ms={a[1]:10.2f} share={100 * a[1] / tot:5.1f}% "
                        f"avg_ms={a[1] / a[0]:8.3f}\n")
            passes = sum(a[1] for k, a in agg.items() if k.startswith("ptsbe_pass"))
            f.write(f"pass kernels share of all device time: {100 * passes / tot:.1f}%\n")
    pf = G / f"pass_dram_{d}_{tag}.csv"
    if pf.exists():
        per = collections.OrderedDict()
        for h, r in rows_of(pf):
            key = r[h["ID"]]
            e = per.setdefault(key, {"name": r[h["Kernel Name"]], "read": 0.0, "write": 0.0, "ms": 0.0})
            m, v, u = r[h["Metric Name"]], float(r[h["Metric Value"]].replace(",", "")), r[h["Metric Unit"]]
            if m == "dram__bytes_read.sum":
                e["read"] = v * BYTES.get(u, 1)
            elif m == "dram__bytes_write.sum":
                e["write"] = v * BYTES.get(u, 1)
            elif m == "gpu__time_duration.sum":
                e["ms"] = v * UNIT.get(u, 1.0)
        launches = list(per.values())
        by = [e["read"] + e["write"] for e in launches]
        shutil.copy(pf, f"{out}_pass_dram_config4_{d}.csv")
        n_q = 28
        amp = 16 if d == "c128" else 8
        traffic = {
            "per_launch_dram_bytes": sum(by) / len(by),
            "launches": len(by),
            "per_pass_dram_bytes": by,
            "per_pass_ncu_ms": [e["ms"] for e in launches],
            "kernels": [e["name"] for e in launches],
            "config": 4, "batch_per_gpu": batch[d], "dtype": d,
            "note": f"algorithmic bytes per launch = 2 * E * 2^{n_q} * {amp} B (E = launch entries incl. the trunk)",
            "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k "
                      f"regex:ptsbe_pass of one bench step after 3 warm-up steps (gpurun tag {tag}; raw CSV "
                      f"{Path(out).name}_pass_dram_config4_{d}.csv)",
        }
        Path(f"profiles/pass_traffic_config4_{d}.json").write_text(json.dumps(traffic, indent=1) + "\n")
        print(d, "passes", len(by), "mean GB/launch", round(traffic["per_launch_dram_bytes"] / 1e9, 2))
