"""PTSBE batched-execution benchmark (BASELINE.json metric: shots/s & trajectories/s; pass GB/s).

One step = one batch of B pre-sampled trajectories of the 28-qubit QEC circuit
(config 4: four [[7,1,3]] Steane blocks, depolarizing + bit-flip on every
target) prepared through the fused device passes and sampled with 10^4 shots
each.  Trajectories are dealt to ranks by id (weak scaling, no collective on
the hot path); every trajectory t keeps seed mix_seed(seed, t).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

The headline is complex128 -- the reference's own arithmetic
(``statevector.py:18-32``); the complex64 engine (north_star's fp32 mode) is
reported beside it under ``"c64"`` in the same line.

value : shots/s of the whole job with inputs resident in HBM (device pointers)
e2e   : the same through the C-ABI with host buffers (H2D of the outcome table,
        D2H of the CSR shot records inside the timed region)

``--impl reference`` times the reference itself (``trajsim`` installed under
``baseline/_ref``; the oracle port only if that install is missing) on the
box's host cores: the op loop of ``prepare_state`` (``execute.py:85-97``) over
a prefix of the same trajectories' op streams, one trajectory per thread, plus
``sample_shots`` at m = 10^4, extrapolated per op kind to the whole stream.
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
# one metric string for both arms (the driver pairs the lines on it)
METRIC = "shots/sec (config 4: 28-qubit QEC circuit, 1e4 shots/trajectory)"


def metric_for(config: int) -> str:
    if config == 5:
        return "shots/sec (config 5: 34-35-qubit QEC state sharded within the trajectory, 1e6 shots/trajectory)"
    return METRIC if config == 4 else f"shots/sec (config {config}, 1e4 shots/trajectory)"
DTYPE_NAME = {"c128": "c128 (complex128, f64 arithmetic)", "c64": "c64 (complex64, f32 arithmetic)"}
# trajectories per step (config 4, prefix-sorted job, 12 timed batches): c128 24 / 28 / 36 ->
# 722 / 747 / 728 K shots/s; c64 48 / 64 / 80 -> 1.76 / 1.77 / 1.75 M
DEFAULT_BATCH = {"c128": 28, "c64": 48}
# trajectories of the whole job (BASELINE.json configs): config 4 = 10^4 trajectories x 10^4 shots
JOB_TRAJECTORIES = {1: 100, 3: 1_000, 4: 10_000}


def workload_config(config: int, world: int) -> dict:
    """The workload description, identical in both arms."""
    return {"workload": "config4 steane_blocks(4): 28 q, 390 ops, 560 sites, probabilistic PTS"
            if config == 4 else f"config{config}",
            "job_trajectories": JOB_TRAJECTORIES.get(config),
            "shots_per_trajectory": SHOTS, "parallelism": f"traj-dp{world}",
            "step": "one batch of the job's trajectories prepared + sampled; timed steps = evenly spaced "
                    "batches of the job's execution order",
            "l2": "inputs larger than L2 (2-4 GiB states)"}


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


def make_workload(config: int, n_traj: int, seed: int, api=None):
    """Circuit + the first n_traj accepted probabilistic-PTS specs (cli.py:100 seeding).

    ``api`` is the module whose parser / PTS runs (this package, or the reference
    itself for the reference arm); both give identical specs (bit-exact PTS)."""
    if api is None:
        import paper_2504_16297_b200 as api
    from paper_2504_16297_b200 import workloads
    c = workloads.build(config, api.parse_circuit, api.parse_noise_model, api.attach_noise)
    specs = []
    nsamples = max(64, 3 * n_traj)
    while len(specs) < n_traj:
        specs = api.presample_probabilistic(c, nsamples, SHOTS, api.stream_rng(seed, 2**63))
        nsamples *= 2
    return c, specs[:n_traj]


# ---------------------------------------------------------------- reference CPU path

def load_reference():
    """The reference package from baseline/_ref (unmodified install), else None."""
    ref_dir = REPO / "baseline" / "_ref"
    if not (ref_dir / "trajsim" / "__init__.py").exists():
        return None
    if str(ref_dir) not in sys.path:
        sys.path.insert(0, str(ref_dir))
    try:
        import trajsim
        import trajsim.statevector as sv
    except Exception:   # noqa: BLE001 -- a broken install falls back to the port
        return None
    sv.MAX_QUBITS = max(sv.MAX_QUBITS, 30)   # lifts the 24-q cap
    return trajsim


def reference_op_stream(ref, circuit, spec):
    """prepare_state's op loop (execute.py:85-97) as (category, thunk(state) -> state) items."""
    sv = ref.statevector
    chosen = dict(spec.selections)
    by_pos = circuit.sites_by_position()
    out = []
    for pos, op in enumerate(circuit.ops):
        out.append((("gate", len(op.targets), False), lambda s, op=op: sv.apply_gate(s, op)))
        for site in by_pos.get(pos, ()):
            k = chosen.get(site.site_id, 0)
            ch = circuit.channels[site.channel_id]
            mix = ch.unitary_mixture()
            if mix is not None:
                out.append((("site", len(site.targets), False),
                            lambda s, m=mix.unitaries[k], t=site.targets: sv.apply_matrix(s, m, t)))
            else:
                out.append((("site", len(site.targets), True),
                            lambda s, m=ch.kraus_ops[k], t=site.targets: sv.apply_kraus_normalized(s, m, t)[0]))
    return out


def port_op_stream(circuit, spec):
    """Same loop on the oracle port (only if the reference install is missing)."""
    from oracle import engine as O
    n = circuit.n_qubits
    out = []
    for mat, targets, general in O.op_stream(circuit, spec.selections):
        def f(psi, mat=mat, targets=targets, general=general):
            psi = O.apply_local(psi, mat, targets, n)
            if general:
                psi = psi / np.sqrt(float(np.sum(np.abs(psi) ** 2)))
            return psi
        out.append((("op", len(targets), general), f))
    return out


class CpuReference:
    """The reference's CPU path on host threads, one trajectory per thread.

    Every step each worker applies the next ``ops_per_step`` entries of its
    trajectory's op stream (workers start at evenly spaced points of the
    stream, so 1q/2q gates and noise sites are all sampled), timing each by
    kind (gate / site, arity, renormalising); the last
    step also draws the trajectory's 10^4 shots with the reference's
    ``sample_shots``.  Per-trajectory time = sum over the FULL stream of the
    per-kind mean op time + the sample time; throughput = workers / that.
    """

    def __init__(self, config: int, seed: int, workers: int | None = None):
        self.ref = load_reference()
        api = self.ref
        if api is None:
            import paper_2504_16297_b200 as api
        cores = os.cpu_count() or 1
        try:
            import psutil
            avail = psutil.virtual_memory().available
        except Exception:   # noqa: BLE001
            avail = 64 << 30
        self.c, specs = make_workload(config, max(cores, 1), seed, api=api)
        n = self.c.n_qubits
        state_b = (1 << n) * 16
        mem_workers = max(1, int(avail * 0.7 // (5 * state_b)))   # state + result + numpy temporaries
        self.workers = workers or max(1, min(cores, mem_workers, len(specs)))
        self.kind = "reference" if self.ref is not None else "port"
        self.specs = specs[: self.workers]
        self.cores = cores
        self.seed = seed
        if self.ref is not None:
            self.streams = [reference_op_stream(self.ref, self.c, s) for s in self.specs]
        else:
            self.streams = [port_op_stream(self.c, s) for s in self.specs]
        self.states = None
        # workers start at evenly spaced points of the op stream, so the timed sample mixes
        # the kinds of the whole stream (1q/2q gates, noise sites), not only the first ops
        L = len(self.streams[0])
        self.pos = [(w * L) // self.workers for w in range(self.workers)]
        self.times: dict = {}
        self.t_sample: list = []
        self.blas_limit = None
        if self.workers > 1:     # one BLAS thread per worker: the workers are the parallelism
            try:
                from threadpoolctl import threadpool_limits
                self.blas_limit = threadpool_limits(1)
            except Exception:   # noqa: BLE001
                pass

    def _zero(self):
        n = self.c.n_qubits
        if self.ref is not None:
            return self.ref.statevector.init_zero(n)
        from oracle import engine as O
        return O.zero_state(n)

    def step(self, ops_per_step: int, timed: bool, sample: bool = False) -> float:
        from concurrent.futures import ThreadPoolExecutor
        if self.states is None:
            self.states = [self._zero() for _ in range(self.workers)]

        def work(w):
            rec = []
            st = self.states[w]
            stream = self.streams[w]
            for _ in range(ops_per_step):
                cat, f = stream[self.pos[w] % len(stream)]
                t0 = time.perf_counter()
                st = f(st)
                rec.append((cat, time.perf_counter() - t0))
                self.pos[w] += 1
            ts = None
            if sample:
                t0 = time.perf_counter()
                if self.ref is not None:
                    self.ref.statevector.sample_shots(st, SHOTS, self.ref.stream_rng(self.seed, w))
                else:
                    from oracle import engine as O
                    O.sample(st / np.linalg.norm(st), SHOTS, np.random.default_rng(w), self.c.n_qubits)
                ts = time.perf_counter() - t0
            self.states[w] = st
            return rec, ts

        t0 = time.perf_counter()
        with ThreadPoolExecutor(max_workers=self.workers) as pool:
            res = list(pool.map(work, range(self.workers)))
        wall = time.perf_counter() - t0
        if timed:
            for rec, ts in res:
                for cat, dt in rec:
                    self.times.setdefault(cat, []).append(dt)
                if ts is not None:
                    self.t_sample.append(ts)
        return wall

    def estimate(self) -> dict:
        """Extrapolated per-trajectory time over the full op stream and the resulting rates."""
        all_t = [t for v in self.times.values() for t in v]
        mean_all = float(np.mean(all_t)) if all_t else float("nan")
        per_cat = {cat: float(np.mean(v)) for cat, v in self.times.items()}
        full = self.streams[0]
        t_prep = 0.0
        for cat, _f in full:
            # an untimed kind: nearest timed kind of the same arity, else the overall mean
            t = per_cat.get(cat)
            if t is None:
                same = [v for k, v in per_cat.items() if k[1] == cat[1]]
                t = float(np.mean(same)) if same else mean_all
            t_prep += t
        t_s = float(np.mean(self.t_sample)) if self.t_sample else 0.0
        per_traj = t_prep + t_s
        traj_s = self.workers / per_traj
        kinds = {f"{k[0]}{k[1]}q{'_renorm' if k[2] else ''}": [len(v), round(float(np.mean(v)), 4)]
                 for k, v in self.times.items()}
        return {"traj_s": traj_s, "shots_s": traj_s * SHOTS, "per_traj_s": per_traj, "t_sample_s": t_s,
                "ops_timed": len(all_t), "g_ref": len(full), "kinds": kinds}

    def sample_text(self, est: dict) -> str:
        src = ("trajsim (baseline/_ref, unmodified; MAX_QUBITS raised to 30)" if self.ref is not None
               else "oracle port (reference install missing)")
        return (f"{src}: {est['ops_timed']} timed ops of the prepare_state op loop (each worker a run of "
                f"its trajectory's stream from an evenly spaced start: 1q/2q gates and noise sites, "
                f"complex128) + sample_shots(m=1e4) on "
                f"{self.workers} threads (one trajectory each, {self.cores} host cores), extrapolated per op "
                f"kind to the full stream of G_ref={est['g_ref']} ops; per-kind [count, mean s]: {est['kinds']}")


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cpu = CpuReference(args.config, args.seed)
    ops = max(1, args.ops_per_step)
    for _ in range(args.warmup):             # real warm-up: the same work, untimed
        cpu.step(ops, timed=False)
    walls = []
    for i in range(max(1, args.steps)):
        walls.append(cpu.step(ops, timed=True, sample=(i == max(1, args.steps) - 1)))
    est = cpu.estimate()
    v = est["shots_s"]
    line = {"impl": "reference", "metric": metric_for(args.config), "value": v, "unit": "shots/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(walls)),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": DTYPE_NAME["c128"],
            "data": "synthetic (PTS-sampled Kraus selections of a generated circuit)",
            "config": workload_config(args.config, world),
            "trajectories_per_s": est["traj_s"],
            "cpu_baseline": {"value": v, "unit": "shots/s", "cores": cpu.workers, "kind": cpu.kind,
                             "sample": cpu.sample_text(est)},
            "e2e": {"value": v, "unit": "shots/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- device path

def run_engine_leg(args, dtype: str, batch: int, c, specs_for, dev, world, rank, local, with_e2e=True):
    """Time K steps of one engine (dtype) on this rank; returns the measurements."""
    import torch
    import torch.distributed as dist

    from paper_2504_16297_b200 import _native as N
    from paper_2504_16297_b200.engine import Engine, pcg64_state_words
    from paper_2504_16297_b200.execute import mix_seed
    from paper_2504_16297_b200.program import compile_circuit, prefix_order, selection_matrix

    B, W, K = batch, args.warmup, args.steps
    per_rank = (W + K) * B
    share_ids, share_specs = specs_for()      # this rank's share of the whole job's trajectories
    prog = compile_circuit(c, dtype, tile_bits=args.tile_bits, low_bits=args.low_bits,
                           search_iters=args.search_iters)
    # The job runs its share in batches of B in the order execute_all uses (trajectories with
    # common outcome prefixes side by side: the engine's tree schedule computes a shared prefix
    # once).  A step = one of those batches; the timed steps are K batches evenly spaced over the
    # whole order (an unbiased sample of the job's batches), the warm-up steps W others.
    order = list(range(len(share_specs))) if args.no_prefix_order else prefix_order(prog, share_specs)
    nb = len(order) // B
    timed = sorted({min(nb - 1, int((i + 0.5) * nb / K)) for i in range(K)})
    if nb < W + K or len(timed) < K:
        raise SystemExit(f"job too small for {W} + {K} steps of {B} trajectories ({len(order)} per rank)")
    rest = [j for j in range(nb) if j not in set(timed)]
    warm = [rest[int(i * len(rest) / W)] for i in range(W)]
    pick = [order[j * B + i] for j in warm + timed for i in range(B)]
    ids, specs = [share_ids[i] for i in pick], [share_specs[i] for i in pick]
    steps_info = {"job_trajectories_per_rank": len(order), "batches_per_rank": nb, "timed_batches": timed}
    eng = Engine(c.n_qubits, dtype, batch_cap=B, device=local)
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
        # inputs resident in HBM; the host's own copies of the outcome table / shot counts (it
        # made them) stand in for device read-backs, so the stream never drains between steps
        lo = i * B
        eng.set_host_mirror(sel[lo:lo + B], shots[lo:lo + B])
        eng.run_device(d_sel.data_ptr() + lo * S, B, d_w.data_ptr(), d_s.data_ptr(), mirror=True)
        eng.sample_device(B, d_shots.data_ptr() + lo * 8, rng_mode, d_rng.data_ptr() + lo * 8 * rng_words.shape[1],
                          d_idx.data_ptr(), d_cnt.data_ptr(), d_nu.data_ptr(), mirror=True)

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
    step_ms = e0.elapsed_time(e1)
    ms = max_over_ranks(step_ms)
    total_traj = K * B * world
    out = {"prog": prog, "eng_info": eng.info(), "t_load": t_load, "steps_info": steps_info, "ms": ms,
           "value": total_traj * SHOTS / (ms / 1e3),
           "traj_s": total_traj / (ms / 1e3), "launches": launches, "clocks": clk.summary(),
           "pass_ms": pass_ms, "pass_n": pass_n, "pass_bytes": pass_bytes, "pp_ms": pp_ms, "pp_bytes": pp_bytes,
           "step_ms_local": step_ms, "total_traj": total_traj}

    if with_e2e:
        # e2e: host buffers through the C ABI, copies inside the timed region; the CSR shot
        # records land in pinned host memory (full-speed DMA), allocated once outside
        sel_host = torch.from_numpy(np.ascontiguousarray(sel)).pin_memory().numpy()
        pin_idx = torch.empty(B * SHOTS, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
        pin_cnt = torch.empty(B * SHOTS, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
        barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        h2d = d2h = 0
        for i in range(W, W + K):
            lo = i * B
            w, st = eng.run(sel_host[lo:lo + B])
            o = eng.sample(shots[lo:lo + B], rng_mode, rng_state=rng_words[lo:lo + B].reshape(-1),
                           out=(pin_idx, pin_cnt))
            h2d += sel_host[lo:lo + B].nbytes + shots[lo:lo + B].nbytes + rng_words[lo:lo + B].nbytes
            d2h += w.nbytes + st.nbytes + o.indices.nbytes + o.counts.nbytes + 8 * B
        t1.record(stream)
        barrier()
        ms_e2e = max_over_ranks(t0.elapsed_time(t1))
        out["e2e"] = {"value": total_traj * SHOTS / (ms_e2e / 1e3), "unit": "shots/s",
                      "h2d_bytes_per_step": h2d // K, "d2h_bytes_per_step": d2h // K}
    eng.close()
    del d_sel, d_shots, d_rng, d_w, d_s, d_idx, d_cnt, d_nu
    torch.cuda.empty_cache()
    return out


def roofline_of(leg, dtype: str, batch: int, config: int, K: int):
    hbm, peak_kind = peaks()
    # algorithmic bytes: one read + one write of every state each pass launch processes
    # (2 * E * 2^n * s; E = trajectories + shared trunk in the launch), summed by the engine
    bytes_per_launch = leg["pass_bytes"] / max(leg["pass_n"], 1)
    avg_launch_ms = leg["pass_ms"] / max(leg["pass_n"], 1)
    achieved = bytes_per_launch / (avg_launch_ms / 1e3) / 1e9
    traffic, traffic_src, ratio = None, None, None
    tf = REPO / "profiles" / f"pass_traffic_config{config}_{dtype}.json"
    if tf.exists():   # ncu DRAM bytes / algorithmic bytes of the pass launches (committed capture)
        t = json.loads(tf.read_text())
        if (t.get("config"), t.get("batch_per_gpu"), t.get("dtype")) == (config, batch, dtype) and \
                t.get("dram_over_algorithmic"):
            ratio = float(t["dram_over_algorithmic"])
            traffic, traffic_src = ratio * bytes_per_launch, t["source"]
    return {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
            "traffic": traffic, "traffic_unit": "bytes/launch (dram read+write, ncu)", "traffic_source": traffic_src,
            "traffic_over_algorithmic": ratio,
            "kernel": "ptsbe_pass_<p> (circuit-specialised fused pass kernels, NVRTC sm_100a)",
            "peak_kind": peak_kind, "bytes_per_launch": bytes_per_launch, "avg_launch_ms": avg_launch_ms,
            "pass_share_of_step": leg["pass_ms"] / max(1e-9, leg["step_ms_local"]),
            "per_pass_ms": [round(float(x) / K, 3) for x in leg["pp_ms"]],
            "per_pass_gbs": [round(float(b) / max(float(m), 1e-9) / 1e6, 1)
                             for m, b in zip(leg["pp_ms"], leg["pp_bytes"])]}


# ---------------------------------------------------------------- config 5: sharded state

C5_SHOTS = 1_000_000


def run_config5(args):
    """Config 5: one 34/35-qubit QEC trajectory's state sharded within the
    trajectory.  N = 1: the 34-qubit form (workloads.CONFIG5_34) as two virtual shards of 33
    local qubits on one GPU (2 x 64 GiB at c64); N >= 2: the 35-qubit circuit over N ranks
    (one shard per GPU, the engine's NCCL group: swaps as one all-to-all per swap point).
    A step = one trajectory prepared + 10^6 Philox shots; value = shots/s of the job."""
    import torch
    import torch.distributed as dist

    import paper_2504_16297_b200 as P
    from paper_2504_16297_b200 import workloads
    from paper_2504_16297_b200.execute import mix_seed
    from paper_2504_16297_b200.sharded import (DistributedShards, EngineShardBackend, VirtualShards, plan_sharded,
                                              sharded_selection)
    rank, world, local = dist_env()
    dtype = "c64"
    if world == 1:
        c = workloads.build(workloads.CONFIG5_34, P.parse_circuit, P.parse_noise_model, P.attach_noise)
        k = 1
    else:
        c = workloads.build(5, P.parse_circuit, P.parse_noise_model, P.attach_noise)
        k = world.bit_length() - 1
        if 1 << k != world:
            raise SystemExit("config 5 needs a power-of-two GPU count")
    W, K = args.warmup, args.steps
    specs = [s for s in P.presample_probabilistic(c, 4 * (W + K) + 8, C5_SHOTS, P.stream_rng(args.seed, 2**63))
             if s.selections][:W + K]
    plan = plan_sharded(c, k, dtype=dtype)
    dev = torch.device("cuda", local)
    if world == 1:
        runner = VirtualShards(plan, dtype, batch_cap=1, device=local)
        run = lambda sel: runner.run(sel)                                  # noqa: E731
        sample = lambda shots, seeds: runner.sample(shots, seeds)          # noqa: E731
    else:
        backend = EngineShardBackend(plan, dtype, batch_cap=1, device=local)
        runner = DistributedShards(plan, backend)
        run = lambda sel: runner.run(sel)                                  # noqa: E731
        sample = lambda shots, seeds: runner.sample(shots, seeds)          # noqa: E731

    def step(i):
        run(sharded_selection(plan, [specs[i]]))
        sample([C5_SHOTS], [mix_seed(args.seed, i)])

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
    for i in range(W):
        step(i)
    barrier()
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        for i in range(W, W + K):
            step(i)
        barrier()
        dt = time.perf_counter() - t0
    t = torch.tensor([dt], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dt = float(t.item())
    if rank == 0:
        n = c.n_qubits
        passes = plan.program.n_passes
        bytes_traj = passes * 2 * (1 << n) * 8
        line = {"metric": metric_for(5), "value": K * C5_SHOTS / dt, "unit": "shots/s", "n_gpus": world, "steps": K,
                "warmup": W, "ms_per_step": 1e3 * dt / K, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": DTYPE_NAME[dtype],
                "data": "synthetic (PTS-sampled Kraus selections of a generated circuit)",
                "config": {"workload": f"config5 {'steane_blocks(4, ancillas=6)' if world == 1 else 'steane_blocks(5)'}:"
                                       f" {n} q, {len(c.ops)} ops, state sharded over 2^{k} shards"
                                       f"{' (virtual, one GPU)' if world == 1 else ' (one per GPU, NCCL)'}",
                           "shots_per_trajectory": C5_SHOTS, "parallelism": f"state-shard{1 << k}",
                           "l2": "inputs larger than L2"},
                "engine": {"passes": passes, "swaps": plan.n_swaps, "local_qubits": plan.n_local,
                           "timing": "host wall clock around K device-synchronised steps, max over ranks"},
                "trajectories_per_s": K / dt,
                "traj_roofline_frac": (K / dt) / (peaks()[0] * 1e9 * world / bytes_traj),
                "clocks": clk.summary(),
                "cpu_baseline": {"value": None, "unit": "shots/s", "cores": 0, "kind": "reference",
                                 "sample": "not runnable on CPU: a 34-35 qubit complex128 state is 256-512 GiB "
                                           "(SURVEY 8(d))"}}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=CONFIG)
    ap.add_argument("--batch", type=int, default=None, help="trajectories per step (default per dtype)")
    ap.add_argument("--dtype", default="c128", choices=["c64", "c128"], help="headline arithmetic")
    ap.add_argument("--secondary", default="c64", choices=["c64", "c128", "none"],
                    help="second engine reported in the same line")
    ap.add_argument("--seed", type=int, default=2024)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--ops-per-step", type=int, default=1, help="reference arm: ops per worker per step")
    ap.add_argument("--rng", default="philox", choices=["philox", "pcg64"])
    ap.add_argument("--tile-bits", type=int, default=None, help="fused-pass tile qubits (default: planner's)")
    ap.add_argument("--low-bits", type=int, default=None, help="contiguous low qubits per tile row (default: planner's)")
    ap.add_argument("--search-iters", type=int, default=None, help="layout-search steps of the planner")
    ap.add_argument("--no-prefix-order", action="store_true",
                    help="run trajectories in PTS order instead of grouping common outcome prefixes")
    ap.add_argument("--no-errors", action="store_true",
                    help="analysis only: zero every sampled Kraus selection (all trajectories noiseless)")
    args = ap.parse_args()
    if args.impl == "reference":
        if args.config == 5:
            if dist_env()[0] == 0:
                print(json.dumps({"impl": "reference", "unavailable": "config 5 (34-35 qubits) does not fit a "
                                  "CPU statevector (256-512 GiB at complex128; SURVEY 8(d))"}), flush=True)
            return
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.config == 5:
        run_config5(args)
        return
    dev = torch.device("cuda", local)
    W, K = args.warmup, args.steps
    legs = [args.dtype] + ([args.secondary] if args.secondary not in ("none", args.dtype) else [])
    batches = {d: (args.batch if (args.batch and d == args.dtype) else DEFAULT_BATCH[d]) for d in legs}
    need = max(JOB_TRAJECTORIES.get(args.config, 0), 2 * max(batches.values()) * (W + K) * world)
    c, specs_all = make_workload(args.config, need, args.seed)

    def specs_for():
        # deterministic deal by trajectory id: rank r owns a contiguous block of the job's ids
        per = len(specs_all) // world
        ids = list(range(rank * per, (rank + 1) * per))
        return ids, [specs_all[i] for i in ids]

    res = {}
    for d in legs:
        res[d] = run_engine_leg(args, d, batches[d], c, specs_for, dev, world, rank, local)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    hbm, _ = peaks()
    head = res[args.dtype]
    B = batches[args.dtype]
    amp = 8 if args.dtype == "c64" else 16
    prog = head["prog"]
    # per trajectory: pass 0 writes the state, every later pass reads + writes it, sampling reads it
    traj_bytes = (2 * prog.n_passes - 1) * (1 << c.n_qubits) * amp + (1 << c.n_qubits) * amp + 16 * SHOTS
    line = {
        "metric": metric_for(args.config), "value": head["value"], "unit": "shots/s",
        "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": head["ms"] / K, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": DTYPE_NAME[args.dtype],
        "data": "synthetic (PTS-sampled Kraus selections of a generated circuit)",
        "config": workload_config(args.config, world),
        "engine": {"batch_per_gpu": B, "passes": prog.n_passes, "g_ref": prog.g_ref, "rng": args.rng,
                   "codegen": bool(head["eng_info"]["codegen"]), "program_load_s": round(head["t_load"], 2),
                   "trajectories_timed": head["total_traj"],
                   "execution_order": "PTS order" if args.no_prefix_order else "prefix-sorted (execute_all's)",
                   **head["steps_info"]},
        "trajectories_per_s": head["traj_s"],
        "traj_roofline_frac": head["traj_s"] / (hbm * 1e9 * world / traj_bytes),
        "roofline": roofline_of(head, args.dtype, B, args.config, K),
        "e2e": head["e2e"],
        "gpu_launches": head["launches"],
        "clocks": head["clocks"],
    }
    for d in legs[1:]:
        r = res[d]
        rf = roofline_of(r, d, batches[d], args.config, K)
        line[d] = {"value": r["value"], "unit": "shots/s", "ms_per_step": r["ms"] / K,
                   "trajectories_per_s": r["traj_s"], "e2e": r["e2e"], "batch_per_gpu": batches[d],
                   "passes": r["prog"].n_passes, "gpu_launches": r["launches"], "clocks": r["clocks"],
                   "roofline": {k: rf[k] for k in ("achieved", "peak", "frac", "traffic", "avg_launch_ms",
                                                   "per_pass_ms", "per_pass_gbs", "pass_share_of_step")}}
    if not args.no_cpu and world == 1:   # CPU baseline on rank 0 at N=1 only (bounded sample)
        cpu = CpuReference(args.config, args.seed)
        cpu.step(1, timed=False)
        for i in range(2):
            cpu.step(2, timed=True, sample=(i == 1))
        est = cpu.estimate()
        line["cpu_baseline"] = {"value": est["shots_s"], "unit": "shots/s", "cores": cpu.workers,
                                "kind": cpu.kind, "sample": cpu.sample_text(est)}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
