"""Split an ncu SASS source CSV (tools/ncu_pass_sass.sh) into the hot kernel body and its
out-of-line slow functions: instructions executed, stall samples, top stall reasons."""
import csv, re, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
h = {k: i for i, k in enumerate(rows[1])}
data = rows[2:]
def n(r, k):
    try:
        return float(r[h[k]])
    except (KeyError, ValueError):
        return 0.0
addr = [int(r[h["Address"]], 16) for r in data]
calls = [int(m.group(1), 16) for r in data for m in [re.search(r"CALL.REL.NOINC (0x[0-9a-f]+)", r[h["Source"]])] if m]
first = min(calls) if calls else 1 << 64
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
for name, part in (("hot", [r for r, a in zip(data, addr) if a < first]), ("slow", [r for r, a in zip(data, addr) if a >= first])):
    ex = sum(n(r, "Instructions Executed") for r in part)
    sm = sum(n(r, "Warp Stall Sampling (All Samples)") for r in part)
    st = collections.Counter({k: sum(n(r, k) for r in part) for k in stalls})
    ops = collections.Counter()
    for r in part:
        m = re.match(r"\s*(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", r[h["Source"]])
        if m:
            ops[m.group(1)] += n(r, "Instructions Executed")
    print(f"{name}: inst {ex:.3g}  samples {sm:.3g}  " + " ".join(f"{k[6:]}:{100 * v / max(sm, 1):.0f}%" for k, v in st.most_common(6)))
    print("   executed mix:", " ".join(f"{k}:{100 * v / max(ex, 1):.0f}%" for k, v in ops.most_common(12)))
