"""execute_all + Dataset.write on the GPU box: dataset path timing (native writer vs json.dumps lines).
   python tools/dataset_speed.py [CONFIG] [TRAJECTORIES]"""
import json, sys, tempfile, time
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
from pathlib import Path

import numpy as np

import paper_2504_16297_b200 as P
from paper_2504_16297_b200 import workloads

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
T = int(sys.argv[2]) if len(sys.argv) > 2 else 256
c = workloads.build(cfg, P.parse_circuit, P.parse_noise_model, P.attach_noise)
specs = P.presample_probabilistic(c, T, 10_000, P.stream_rng(1, 2**63))
P.execute_all(c, specs[:2], dtype="c64", rng="philox")          # program load / warm-up
t0 = time.perf_counter()
ds = P.execute_all(c, specs, dtype="c64", rng="philox")
t1 = time.perf_counter()
d = Path(tempfile.mkdtemp())
ds.write(d / "native")
t2 = time.perf_counter()
P.Dataset(ds.manifest, list(ds.records)).write(d / "json")
t3 = time.perf_counter()
same = (d / "native" / "records.jsonl").read_bytes() == (d / "json" / "records.jsonl").read_bytes()
print(json.dumps({"config": cfg, "trajectories": len(specs), "records": len(ds.records),
                  "execute_all_s": round(t1 - t0, 3), "write_native_s": round(t2 - t1, 3),
                  "write_json_s_incl_record_objects": round(t3 - t2, 3), "identical": same}))
