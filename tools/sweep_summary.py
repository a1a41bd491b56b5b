import sys, json
for l in open(sys.argv[1]):
    if l.startswith("=="):
        print(l.strip()); continue
    try:
        d = json.loads(l)
    except ValueError:
        print("   ", l.strip()[:200]); continue
    print("   value %.0f e2e %.0f frac %.3f ms/step %.1f passes %s" % (d["value"], d["e2e"]["value"], d["roofline"]["frac"],
                                                                   d["ms_per_step"], d["config"]["passes"]))
    r = d["roofline"]
    if "per_pass_ms" in r:
        print("   per-pass ms  ", " ".join(f"{x:6.1f}" for x in r["per_pass_ms"]))
        print("   per-pass GB/s", " ".join(f"{x:6.0f}" for x in r["per_pass_gbs"]))
