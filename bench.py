"""PTSBE batched-execution benchmark (BASELINE.json metric: shots/s & trajectories/s; pass GB/s).

One step = one batch of B pre-sampled trajectories of the 28-qubit QEC circuit
(config 4: four [[7,1,3]] Steane blocks, depolarizing + bit-flip on every
target) prepared through the fused device passes and sampled with 10^4 shots
each.  Trajectories are dealt to ranks by id (weak scaling, no collective on
the hot path); every trajectory t keeps seed mix_seed(seed, t).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

value : shots/s of the whole job with inputs resident in HBM (device pointers)
e2e   : the same through the C-ABI with host buffers (H2D of the outcome table,
        D2H of the CSR shot records inside the timed region)
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

CONFIG = 4
SHOTS = 10_000


def peaks():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, ValueError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def make_workload(config: int, n_traj: int, seed: int):
    import paper_2504_16297_b200 as P
    from paper_2504_16297_b200 import workloads
    from paper_2504_16297_b200.execute import stream_rng
    c = workloads.build(config, P.parse_circuit, P.parse_noise_model, P.attach_noise)
    rng = stream_rng(seed, 2**63)            # cli.py:100 convention
    specs = []
    nsamples = max(64, 3 * n_traj)
    while len(specs) < n_traj:
        specs = P.presample_probabilistic(c, nsamples, SHOTS, rng)
        nsamples *= 2
        rng = stream_rng(seed, 2**63)
    return c, specs[:n_traj]


def cpu_port_rate(c, specs, budget_s: float, workers: int = 1):
    """Oracle (numpy restatement of the reference hot path) on a bounded prefix.

    Times ``k`` ops of the op stream per trajectory (mix of gates and sites, as
    execute.py:85-97 applies them) plus one sample_shots at the full m, and
    extrapolates per-trajectory time = t_op * G_ref + t_sample.
    """
    from concurrent.futures import ThreadPoolExecutor

    from oracle import engine as O
    n = c.n_qubits
    g_ref = len(c.ops) + len(c.sites)

    def one(spec):
        psi = O.zero_state(n)
        t0 = time.perf_counter()
        done = 0
        for mat, targets, general in O.op_stream(c, spec.selections):
            psi = O.apply_local(psi, mat, targets, n)
            if general:
                r = float(np.sum(np.abs(psi) ** 2))
                psi = psi / np.sqrt(r)
            done += 1
            if time.perf_counter() - t0 > budget_s * 0.6:
                break
        t_op = (time.perf_counter() - t0) / done
        t1 = time.perf_counter()
        psi /= np.linalg.norm(psi)
        O.sample(psi, SHOTS, np.random.default_rng(0), n)
        t_s = time.perf_counter() - t1
        return t_op, t_s, done

    with ThreadPoolExecutor(max_workers=workers) as pool:
        res = list(pool.map(one, specs[:workers]))
    t_op = float(np.mean([r[0] for r in res]))
    t_s = float(np.mean([r[1] for r in res]))
    per_traj = t_op * g_ref + t_s
    traj_s = workers / per_traj
    return {"traj_s": traj_s, "shots_s": traj_s * SHOTS, "t_op_s": t_op, "t_sample_s": t_s,
            "ops_timed": int(sum(r[2] for r in res)), "g_ref": g_ref}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    c, specs = make_workload(args.config, 8, args.seed)
    import psutil
    cores = os.cpu_count() or 1
    mem = psutil.virtual_memory().available
    state_b = (1 << c.n_qubits) * 16
    workers = max(1, min(cores, int(mem * 0.3 // (4 * state_b)), 4))
    vals = []
    for _ in range(args.warmup and 0):
        pass
    for step in range(max(1, args.steps)):
        r = cpu_port_rate(c, specs, budget_s=max(4.0, 20.0 / max(1, args.steps)), workers=workers)
        vals.append(r["shots_s"])
    v = float(np.median(vals))
    line = {"impl": "reference", "metric": "shots/sec (config 4, 28 q, 1e4 shots/trajectory)", "value": v,
            "unit": "shots/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128 (f64)",
            "data": "synthetic",
            "config": {"workload": "config4 steane_blocks(4): 28 q, 390 ops, 560 sites, 1e4 shots/traj"},
            "trajectories_per_s": r["traj_s"],
            "cpu_baseline": {"value": v, "unit": "shots/s", "cores": workers, "kind": "port",
                             "sample": f"{r['ops_timed']} ops of the op stream + one 1e4-shot sample per "
                                       f"trajectory on {workers} threads, extrapolated to G_ref={r['g_ref']} ops"},
            "e2e": {"value": v, "unit": "shots/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=CONFIG)
    ap.add_argument("--batch", type=int, default=48)
    ap.add_argument("--dtype", default="c64", choices=["c64", "c128"])
    ap.add_argument("--seed", type=int, default=2024)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--rng", default="philox", choices=["philox", "pcg64"])
    ap.add_argument("--tile-bits", type=int, default=None, help="fused-pass tile qubits (default: planner's)")
    ap.add_argument("--low-bits", type=int, default=None, help="contiguous low qubits per tile row (default: planner's)")
    ap.add_argument("--search-iters", type=int, default=None, help="layout-search steps of the planner")
    ap.add_argument("--no-errors", action="store_true",
                    help="analysis only: zero every sampled Kraus selection (all trajectories noiseless)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    from paper_2504_16297_b200 import _native as N
    from paper_2504_16297_b200.engine import Engine, pcg64_state_words
    from paper_2504_16297_b200.execute import mix_seed
    from paper_2504_16297_b200.program import compile_circuit, selection_matrix

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    B, W, K = args.batch, args.warmup, args.steps
    per_rank = (W + K) * B
    c, specs_all = make_workload(args.config, per_rank * world, args.seed)
    # deterministic deal by trajectory id: rank r owns ids [r*per_rank, (r+1)*per_rank)
    ids = list(range(rank * per_rank, (rank + 1) * per_rank))
    specs = [specs_all[i] for i in ids]
    prog = compile_circuit(c, args.dtype, tile_bits=args.tile_bits, low_bits=args.low_bits,
                           search_iters=args.search_iters)
    eng = Engine(c.n_qubits, args.dtype, batch_cap=B, device=local)
    t_load = time.perf_counter()
    eng.load_program(prog)          # plans phases, generates + NVRTC-compiles the pass kernels
    t_load = time.perf_counter() - t_load
    sel = selection_matrix(prog, specs)
    if args.no_errors:
        sel[:] = 0
    shots = np.full(per_rank, SHOTS, dtype=np.int64)
    if args.rng == "philox":
        rng_mode = N.RNG_PHILOX
        rng_words = np.array([mix_seed(args.seed, t) for t in ids], dtype=np.uint64).reshape(per_rank, 1)
    else:
        rng_mode = N.RNG_PCG64
        rng_words = np.stack([pcg64_state_words(mix_seed(args.seed, t)) for t in ids])
    dev = torch.device("cuda", local)
    # value path: inputs resident in HBM
    d_sel = torch.from_numpy(sel).to(dev)
    d_shots = torch.from_numpy(shots).to(dev)
    d_rng = torch.from_numpy(rng_words.view(np.int64)).to(dev)
    d_w = torch.empty(B, dtype=torch.float64, device=dev)
    d_s = torch.empty(B, dtype=torch.int32, device=dev)
    d_idx = torch.empty(B * SHOTS, dtype=torch.int64, device=dev)
    d_cnt = torch.empty(B * SHOTS, dtype=torch.int32, device=dev)
    d_nu = torch.empty(B, dtype=torch.int64, device=dev)
    S = sel.shape[1]
    stream = torch.cuda.ExternalStream(eng.stream, device=dev)

    def step_device(i):
        lo = i * B
        eng.run_device(d_sel.data_ptr() + lo * S, B, d_w.data_ptr(), d_s.data_ptr())
        eng.sample_device(B, d_shots.data_ptr() + lo * 8, rng_mode, d_rng.data_ptr() + lo * 8 * rng_words.shape[1],
                          d_idx.data_ptr(), d_cnt.data_ptr(), d_nu.data_ptr())

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for i in range(W):
        step_device(i)
    barrier()
    eng.profile(True)
    l0 = eng.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for i in range(W, W + K):
            step_device(i)
        e1.record(stream)
        barrier()
    launches = eng.launches - l0
    pass_ms, pass_n, pass_bytes = eng.profile_read()
    pp_ms, pp_bytes = eng.profile_passes()
    eng.profile(False)
    ms = max_over_ranks(e0.elapsed_time(e1))
    total_traj = K * B * world
    value = total_traj * SHOTS / (ms / 1e3)

    # e2e: host buffers through the C ABI, copies inside the timed region
    sel_host = np.ascontiguousarray(sel)
    barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    h2d = d2h = 0
    for i in range(W, W + K):
        lo = i * B
        w, st = eng.run(sel_host[lo:lo + B])
        out = eng.sample(shots[lo:lo + B], rng_mode, rng_state=rng_words[lo:lo + B].reshape(-1))
        h2d += sel_host[lo:lo + B].nbytes + shots[lo:lo + B].nbytes + rng_words[lo:lo + B].nbytes
        d2h += w.nbytes + st.nbytes + out.indices.nbytes + out.counts.nbytes + 8 * B
    t1.record(stream)
    barrier()
    ms_e2e = max_over_ranks(t0.elapsed_time(t1))
    e2e = total_traj * SHOTS / (ms_e2e / 1e3)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    hbm, peak_kind = peaks()
    amp = 8 if args.dtype == "c64" else 16
    # algorithmic bytes: one read + one write of every state each pass launch processes
    # (2 * E * 2^n * s; E = trajectories + shared trunk in the launch), summed by the engine
    bytes_per_launch = pass_bytes / max(pass_n, 1)
    avg_launch_ms = pass_ms / max(pass_n, 1)
    achieved = bytes_per_launch / (avg_launch_ms / 1e3) / 1e9
    traffic, traffic_src = None, None
    tf = REPO / "profiles" / "pass_traffic_config4.json"
    if tf.exists():   # ncu DRAM bytes per pass launch of the same workload (committed capture)
        t = json.loads(tf.read_text())
        if (t.get("config"), t.get("batch_per_gpu"), t.get("dtype"), t.get("launches")) == \
                (args.config, B, args.dtype, prog.n_passes):
            traffic, traffic_src = t["per_launch_dram_bytes"], t["source"]
            if not traffic == traffic:   # nan counters: report none
                traffic, traffic_src = None, None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": traffic, "traffic_unit": "bytes/launch (dram read+write, ncu)", "traffic_source": traffic_src,
                "kernel": "pass_kernel", "peak_kind": peak_kind,
                "bytes_per_launch": bytes_per_launch, "avg_launch_ms": avg_launch_ms,
                "pass_share_of_step": pass_ms / max(1e-9, e0.elapsed_time(e1)),
                "per_pass_ms": [round(float(x) / K, 3) for x in pp_ms],
                "per_pass_gbs": [round(float(b) / max(float(m), 1e-9) / 1e6, 1) for m, b in zip(pp_ms, pp_bytes)]}
    traj_bytes = prog.n_passes * 2 * (1 << c.n_qubits) * amp + (1 << c.n_qubits) * amp + 16 * SHOTS
    line = {
        "metric": "shots/sec (config 4: 28 q QEC, 1e4 shots/trajectory)", "value": value, "unit": "shots/s",
        "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": ms / K, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c64 (f32 complex)" if args.dtype == "c64" else "c128 (f64 complex)",
        "data": "synthetic (PTS-sampled Kraus selections of a generated circuit)",
        "config": {"workload": "config4 steane_blocks(4): 28 q, %d ops, %d sites" % (len(c.ops), len(c.sites)),
                   "batch_per_gpu": B, "shots_per_trajectory": SHOTS, "passes": prog.n_passes, "g_ref": prog.g_ref,
                   "rng": args.rng, "l2": "inputs larger than L2 (2 GiB states)", "parallelism": f"traj-dp{world}",
                   "codegen": bool(eng.info()["codegen"]), "program_load_s": round(t_load, 2)},
        "trajectories_per_s": total_traj / (ms / 1e3),
        "traj_roofline_frac": (total_traj / (ms / 1e3)) / (hbm * 1e9 * world / traj_bytes),
        "roofline": roofline,
        "e2e": {"value": e2e, "unit": "shots/s", "h2d_bytes_per_step": h2d // K, "d2h_bytes_per_step": d2h // K},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if not args.no_cpu and world == 1:   # CPU baseline on rank 0 at N=1 only
        r = cpu_port_rate(c, specs, budget_s=15.0, workers=1)
        line["cpu_baseline"] = {"value": r["shots_s"], "unit": "shots/s", "cores": 1, "kind": "port",
                                "sample": f"{r['ops_timed']} ops of one trajectory's op stream + one 1e4-shot "
                                          f"sample (complex128 numpy, as the reference), extrapolated to "
                                          f"G_ref={r['g_ref']} ops"}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
