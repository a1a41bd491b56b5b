"""Trajectory parallelism across GPUs (one process per GPU).

Trajectories are independent, so the hot path has NO collective: rank r takes a
deterministic block of trajectory ids, prepares and samples them on its own
GPU (``execute.run_specs``), and the CSR shot records are merged on rank 0 by
trajectory id after the last batch.  Every trajectory keeps its seed
``mix_seed(master_seed, t)`` whatever rank runs it, so the merged dataset is
byte-identical for any GPU count (the reference's determinism promise across
worker counts, ``execute.py:1-5``, ``test_acceptance.py:240-264``).

The only communication is the final ``gather_object`` of per-rank results
(torch.distributed; NCCL or gloo), outside the timed hot path.
"""

from __future__ import annotations

import numpy as np

from .execute import BatchOutput


def deal(n_traj: int, world: int, rank: int) -> list:
    """Contiguous, balanced block of trajectory ids owned by ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world {world}")
    base, extra = divmod(n_traj, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return list(range(lo, hi))


def merge(parts) -> BatchOutput:
    """Merge per-rank (ids, BatchOutput) pairs into one output ordered by trajectory id."""
    parts = [(list(ids), out) for ids, out in parts if len(ids)]
    if not parts:
        z = np.zeros(0)
        return BatchOutput(z, np.zeros(0, np.int32), np.zeros(0, np.uint64), np.zeros(0, np.uint32),
                           np.zeros(1, np.int64), z, z)
    all_ids = [t for ids, _ in parts for t in ids]
    T = max(all_ids) + 1
    if sorted(all_ids) != list(range(T)):
        raise ValueError("ranks did not cover the trajectory ids exactly once")
    weights = np.zeros(T)
    status = np.zeros(T, dtype=np.int32)
    prep = np.zeros(T)
    samp = np.zeros(T)
    nuniq = np.zeros(T, dtype=np.int64)
    chunks = [None] * T
    for ids, out in parts:
        for j, t in enumerate(ids):
            weights[t] = out.weights[j]
            status[t] = out.status[j]
            prep[t] = out.prep_time[j]
            samp[t] = out.sample_time[j]
            lo, hi = int(out.offsets[j]), int(out.offsets[j + 1])
            chunks[t] = (out.indices[lo:hi], out.counts[lo:hi])
            nuniq[t] = hi - lo
    off = np.zeros(T + 1, dtype=np.int64)
    np.cumsum(nuniq, out=off[1:])
    idx = np.concatenate([c[0] for c in chunks]) if T else np.zeros(0, np.uint64)
    cnt = np.concatenate([c[1] for c in chunks]) if T else np.zeros(0, np.uint32)
    return BatchOutput(weights, status, idx.astype(np.uint64), cnt.astype(np.uint32), off, prep, samp)


def run_distributed(circuit, specs, master_seed: int = 0, dtype: str = "c128", rng: str = "pcg64",
                    runner=None, group=None, device=None):
    """Run this rank's block of ``specs`` and gather everything on rank 0.

    Returns the merged ``BatchOutput`` on rank 0 and ``None`` elsewhere.
    ``runner(circuit, specs, master_seed, dtype, rng, ids)`` defaults to the
    device engine (``execute.run_specs``); tests inject a CPU stand-in.
    """
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    ids = deal(len(specs), world, rank)
    if runner is None:
        from .execute import run_specs

        def runner(c, s, m, d, r, i):
            return run_specs(c, s, m, d, r, ids=i, device=device if device is not None else 0)
    local = runner(circuit, [specs[t] for t in ids], master_seed, dtype, rng, ids) if ids else None
    if world == 1:
        return merge([(ids, local)])
    gathered = [None] * world if rank == 0 else None
    dist.gather_object((ids, local), gathered, dst=dist.get_global_rank(group, 0) if group else 0, group=group)
    if rank != 0:
        return None
    return merge([(i, o) for i, o in gathered if o is not None])


def execute_all_distributed(circuit, specs, master_seed: int = 0, meta: dict | None = None, *,
                            dtype: str = "c128", rng: str = "pcg64", runner=None, group=None, device=None):
    """``execute_all`` over all ranks: the merged Dataset on rank 0, ``None`` elsewhere.

    Same rows, manifest and ``records.jsonl`` bytes as a single-process
    ``execute_all`` of the same specs (ref ``execute.py:130-178``; output
    independent of the worker count, ``execute.py:1-5``).
    """
    import time

    from .execute import dataset_from_output, validate_spec

    specs = list(specs)
    for spec in specs:
        validate_spec(circuit, spec)
    start = time.perf_counter()
    out = run_distributed(circuit, specs, master_seed, dtype, rng, runner=runner, group=group, device=device)
    if out is None:
        return None
    return dataset_from_output(circuit, specs, out if specs else None, master_seed=master_seed, meta=meta,
                               start=start)
