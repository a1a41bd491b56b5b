"""Host PTS overlapped with device batches on config 3 (20 q, 10^4 shots
per trajectory): trajectories/s of
  seq   : presample_probabilistic, then execute_all (PTS and device one after the other)
  pipe  : presample_and_execute (PTS blocks + batch inputs on a host thread while batches run)
  dev   : the device-resident rate of the same batches (engine only, inputs in HBM)
  python tools/pipeline_speed.py [--nsamples N] [--dtype c64] [--rng philox]"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2504_16297_b200 as P  # noqa: E402
from paper_2504_16297_b200 import workloads  # noqa: E402
from paper_2504_16297_b200.execute import execute_all, get_engine, presample_and_execute, run_specs, stream_rng  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--nsamples", type=int, default=2000)
ap.add_argument("--shots", type=int, default=10_000)
ap.add_argument("--dtype", default="c64")
ap.add_argument("--rng", default="philox")
ap.add_argument("--batch", type=int, default=256)
a = ap.parse_args()
c = workloads.build(a.config, P.parse_circuit, P.parse_noise_model, P.attach_noise)
kw = dict(dtype=a.dtype, rng=a.rng)
# warm-up: program load + NVRTC
specs = P.presample_probabilistic(c, 200, a.shots, stream_rng(1, 2**63))
run_specs(c, specs, 1, batch=a.batch, **kw)
res = {"config": a.config, "nsamples": a.nsamples, "shots": a.shots, "dtype": a.dtype, "rng": a.rng}
t0 = time.perf_counter()
specs = P.presample_probabilistic(c, a.nsamples, a.shots, stream_rng(3, 2**63))
t1 = time.perf_counter()
ds = execute_all(c, specs, master_seed=3, **kw)
t2 = time.perf_counter()
res.update(trajectories=len(specs), pts_s=t1 - t0, execute_s=t2 - t1, seq_traj_s=len(specs) / (t2 - t0))
t0 = time.perf_counter()
specs2, ds2 = presample_and_execute(c, a.nsamples, a.shots, stream_rng(3, 2**63), master_seed=3, batch=a.batch, **kw)
t1 = time.perf_counter()
res.update(pipe_s=t1 - t0, pipe_traj_s=len(specs2) / (t1 - t0), same_specs=specs2 == specs)
# device-only: the same batches through the device-pointer engine path (inputs resident)
import torch  # noqa: E402
from paper_2504_16297_b200 import _native as N  # noqa: E402
from paper_2504_16297_b200.execute import mix_seed  # noqa: E402
from paper_2504_16297_b200.program import selection_matrix  # noqa: E402
eng = get_engine(c, a.dtype, want=a.batch)
B = min(eng.cap, a.batch)
sel = selection_matrix(eng.program, specs)
shots = np.array([s.shots for s in specs], dtype=np.int64)
seeds = np.array([mix_seed(3, t) for t in range(len(specs))], dtype=np.uint64)
dev = torch.device("cuda", 0)
d_sel, d_shots, d_rng = (torch.from_numpy(x).to(dev) for x in (sel, shots, seeds.view(np.int64)))
d_w = torch.empty(B, dtype=torch.float64, device=dev)
d_s = torch.empty(B, dtype=torch.int32, device=dev)
d_idx = torch.empty(B * a.shots, dtype=torch.int64, device=dev)
d_cnt = torch.empty(B * a.shots, dtype=torch.int32, device=dev)
d_nu = torch.empty(B, dtype=torch.int64, device=dev)
torch.cuda.synchronize()
t0 = time.perf_counter()
for lo in range(0, len(specs), B):
    hi = min(len(specs), lo + B)
    eng.set_host_mirror(sel[lo:hi], shots[lo:hi])
    eng.run_device(d_sel.data_ptr() + lo * sel.shape[1], hi - lo, d_w.data_ptr(), d_s.data_ptr(), mirror=True)
    eng.sample_device(hi - lo, d_shots.data_ptr() + lo * 8, N.RNG_PHILOX, d_rng.data_ptr() + lo * 8,
                      d_idx.data_ptr(), d_cnt.data_ptr(), d_nu.data_ptr(), mirror=True)
eng.synchronize()
t1 = time.perf_counter()
res.update(dev_s=t1 - t0, dev_traj_s=len(specs) / (t1 - t0))
res["pipe_over_dev"] = res["pipe_traj_s"] / res["dev_traj_s"]
res["seq_over_dev"] = res["seq_traj_s"] / res["dev_traj_s"]
print(json.dumps(res))
