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
batch = {"c128": int(sys.argv[3]) if len(sys.argv) > 3 else 28, "c64": int(sys.argv[4]) if len(sys.argv) > 4 else 48}
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
        # the engine's own launch log of the same process: (pass, entries, algorithmic bytes)
        ll = G / f"launchlog_{d}_{tag}.txt"
        alg = [tuple(float(x) for x in line.split()) for line in open(ll)] if ll.exists() else []
        m = min(len(alg), len(by))
        if m:
            shutil.copy(ll, f"{out}_launchlog_config4_{d}.txt")
        ratio = sum(by[:m]) / sum(a[2] for a in alg[:m]) if m else None
        per_pass = {}
        for (p_, e_, a_), b_ in zip(alg[:m], by[:m]):
            x = per_pass.setdefault(int(p_), [0.0, 0.0])
            x[0] += b_
            x[1] += a_
        traffic = {
            "dram_over_algorithmic": ratio,
            "per_pass_dram_over_algorithmic": {k: v[0] / v[1] for k, v in sorted(per_pass.items())},
            "launches_matched": m,
            "per_launch_dram_bytes": sum(by) / len(by),
            "launches": len(by),
            "config": 4, "batch_per_gpu": batch[d], "dtype": d,
            "note": "algorithmic bytes per launch = 2 * E * 2^n * s (E = launch entries of the tree schedule); "
                    "bench.py reports traffic = dram_over_algorithmic x its own algorithmic bytes per launch",
            "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k "
                      f"regex:ptsbe_pass over every pass launch of a short bench run, matched in order with the "
                      f"engine's PTSBE_LAUNCH_LOG of the same process (gpurun tag {tag}; raw files "
                      f"{Path(out).name}_pass_dram_config4_{d}.csv, {Path(out).name}_launchlog_config4_{d}.txt)",
        }
        Path(f"profiles/pass_traffic_config4_{d}.json").write_text(json.dumps(traffic, indent=1) + "\n")
        print(d, "launches", len(by), "matched", m, "dram / algorithmic", ratio)
