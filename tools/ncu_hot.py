"""Hot source lines / SASS of an ncu report: python tools/ncu_hot.py rep [kernel-substring] [n]"""
import csv, subprocess, sys
rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else ""
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"] +
                     (["-k", kern] if kern else []), capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur_file = None
lines = []   # (file, line, src, samples, inst)
sass = []
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or len(r) < 8:
        continue
    def num(v):
        try:
            return float(v)
        except ValueError:
            return 0.0
    samp = int(num(r[hdr["Warp Stall Sampling (All Samples)"]]))
    inst = int(num(r[hdr["Instructions Executed"]]))
    if r[0]:
        lines.append((samp, inst, cur_file, r[0], r[1][:110]))
    else:
        sass.append((samp, inst, r[3][:60]))
tot_s = sum(x[0] for x in lines) or 1
tot_i = sum(x[1] for x in lines) or 1
print(f"total samples {tot_s}, warp-inst {tot_i}")
for s, i, f, ln, src in sorted(lines, reverse=True)[:n]:
    print(f"{100*s/tot_s:5.1f}% samp {100*i/tot_i:5.1f}% inst  {f}:{ln}  {src}")
