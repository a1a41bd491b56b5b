"""Config 5 on ONE B200: the 34-qubit QEC circuit (workloads.CONFIG5_34: four Steane blocks
+ six syndrome ancillas) as a 2-shard virtual sharded state (2 x 64 GiB at c64), one
trajectory with 10^6 Philox shots -- checked against the unsharded engine (128 GiB) on a
random subset of 2^20 amplitudes, timed per phase.

  python tools/config5.py [--out gpurun_out/config5.json]

Used by tests/test_config5.py (assertions) and for the profiles/ record (timings)."""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def logical_to_shard(logical: np.ndarray, plan):
    """(shard, local physical index) of logical basis indices under the plan's final layout."""
    shard = np.zeros(logical.shape, dtype=np.int64)
    local = np.zeros(logical.shape, dtype=np.uint64)
    for q, (kind, bit) in plan.final_map.items():
        v = (logical >> np.uint64(q)) & np.uint64(1)
        if kind == "L":
            local |= v << np.uint64(bit)
        else:
            shard |= v.astype(np.int64) << bit
    return shard, local


def run(shots: int = 1_000_000, subset: int = 1 << 20, dtype: str = "c64", seed: int = 5):
    import paper_2504_16297_b200 as P
    from paper_2504_16297_b200 import workloads
    from paper_2504_16297_b200.engine import Engine
    from paper_2504_16297_b200.execute import mix_seed
    from paper_2504_16297_b200.program import compile_circuit, selection_matrix
    from paper_2504_16297_b200.sharded import VirtualShards, plan_sharded, sharded_selection

    c = workloads.build(workloads.CONFIG5_34, P.parse_circuit, P.parse_noise_model, P.attach_noise)
    n = c.n_qubits
    spec = next(s for s in P.presample_probabilistic(c, 50, shots, np.random.default_rng(seed)) if s.selections)
    rng = np.random.default_rng(1)
    logical = rng.choice(1 << n, size=subset, replace=False).astype(np.uint64)
    out = {"workload": f"config5-34q: steane_blocks(4, ancillas=6), {n} q, {len(c.ops)} ops, {len(c.sites)} sites",
           "dtype": dtype, "shots": shots, "selections": len(spec.selections)}
    # unsharded reference on the same GPU (128 GiB at c64), identity layout
    t0 = time.perf_counter()
    prog = compile_circuit(c, dtype, search_iters=0)
    with Engine(n, dtype, batch_cap=1) as eng:
        eng.load_program(prog)
        t1 = time.perf_counter()
        w_ref, st_ref = eng.run(selection_matrix(prog, [spec]))
        out["unsharded_run_s"] = time.perf_counter() - t1
        out["unsharded_passes"] = prog.n_passes
        ref = eng.gather(0, logical).astype(np.complex128)
        ref_total = int(eng.norm_totals(1)[0])
    out["unsharded_total_s"] = time.perf_counter() - t0
    # 2 virtual shards of 33 local qubits
    plan = plan_sharded(c, 1, dtype=dtype)
    vs = VirtualShards(plan, dtype, batch_cap=1)
    try:
        sel = sharded_selection(plan, [spec])
        t1 = time.perf_counter()
        w, st = vs.run(sel)
        out["sharded_run_s"] = time.perf_counter() - t1
        out["sharded_passes"] = plan.program.n_passes
        out["swaps"] = plan.n_swaps
        shard, local = logical_to_shard(logical, plan)
        got = np.empty(subset, dtype=np.complex128)
        for s in range(1 << plan.k):
            m = shard == s
            got[m] = vs.engines[s].gather(0, local[m])
        totals = [int(e.norm_totals(1)[0]) for e in vs.engines]
        t1 = time.perf_counter()
        res = vs.sample([shots], [mix_seed(seed, 0)])
        out["sample_s"] = time.perf_counter() - t1
        idx, cnt = res[0]
        sh, lo = logical_to_shard(idx, plan)
        amp_hit = np.concatenate([vs.engines[s].gather(0, lo[sh == s]) for s in range(1 << plan.k)])
    finally:
        vs.close()
    out["subset_rel_l2"] = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
    out["weights"] = [float(w_ref[0]), float(w[0])]
    out["status"] = [int(st_ref[0]), int(st[0])]
    out["norm_total_unsharded"] = ref_total / 2.0 ** 62
    out["norm_total_sharded"] = sum(totals) / 2.0 ** 62
    out["shots_drawn"] = int(cnt.sum())
    out["distinct_outcomes"] = int(idx.size)
    out["min_prob_of_sampled"] = float(np.min(np.abs(amp_hit) ** 2)) if amp_hit.size else None
    out["sorted_unique"] = bool(np.all(np.diff(idx.astype(np.int64)) > 0))
    bytes_pass = 2 * (1 << n) * (8 if dtype == "c64" else 16)
    out["sharded_pass_gbs"] = bytes_pass * out["sharded_passes"] / out["sharded_run_s"] / 1e9
    out["unsharded_pass_gbs"] = bytes_pass * out["unsharded_passes"] / out["unsharded_run_s"] / 1e9
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--shots", type=int, default=1_000_000)
    a = ap.parse_args()
    r = run(a.shots)
    print(json.dumps(r))
    if a.out:
        Path(a.out).write_text(json.dumps(r, indent=1) + "\n")
