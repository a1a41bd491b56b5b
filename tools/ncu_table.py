"""Per-kernel table from an ncu raw CSV (ncu -i rep --page raw --csv): time, DRAM bytes, achieved GB/s,
issue activity, top stall reasons.   python tools/ncu_table.py raw.csv"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = {k: i for i, k in enumerate(rows[0])}
units = rows[1]
def f(r, k):
    try:
        v = float(r[h[k]].replace(",", ""))
    except (KeyError, ValueError):
        return float("nan")
    u = units[h[k]]
    return v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "Tbyte": 1e12,
                "msecond": 1e-3, "usecond": 1e-6, "nsecond": 1e-9, "second": 1, "ms": 1e-3, "us": 1e-6, "ns": 1e-9,
                "s": 1}.get(u, 1)
stall = [k for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
print(f"{'kernel':16s} {'ms':>7s} {'GB':>6s} {'GB/s':>6s} {'dram%':>5s} {'issue%':>6s} {'warps%':>6s} {'inst(M)':>8s} {'bankc%':>6s}  top stalls")
for r in rows[2:]:
    t = f(r, "gpu__time_duration.sum")
    by = f(r, "dram__bytes_read.sum") + f(r, "dram__bytes_write.sum")
    st = sorted(((f(r, k), k.replace("smsp__pcsamp_warps_issue_stalled_", "")) for k in stall), reverse=True)
    tot = sum(v for v, _ in st) or 1
    wav = f(r, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")
    bc = f(r, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum")
    print(f"{r[h['Kernel Name']][:16]:16s} {t * 1e3:7.2f} {by / 1e9:6.1f} {by / t / 1e9:6.0f} "
          f"{f(r, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):5.1f} "
          f"{f(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):6.1f} "
          f"{f(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):6.1f} "
          f"{f(r, 'smsp__inst_executed.sum') / 1e6:8.0f} {100 * bc / wav if wav else 0:6.1f}  "
          + " ".join(f"{k}:{100 * v / tot:.0f}" for v, k in st[:5]))
