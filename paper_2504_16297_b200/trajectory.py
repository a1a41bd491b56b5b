"""Conventional trajectory simulation (Algorithm 1) on the device engine.

Mirror of ``pkg/src/trajsim/trajectory.py``: ``select_index`` (also used by the
PTS strategies), ``run_trajectory`` (``:40-70``) and ``sample_conventional``
(``:73-106``, with its dense-ensemble stream order for n <= 8, ``:138-219``).

The reference walks the ops of ONE trajectory with numpy, drawing one uniform
per noise site: a unitary-mixture site picks ``select_index(r, probs)`` from
the channel's fixed probabilities, a general site first computes every
``||K_k psi||^2`` on the current state.  Here the uniforms are drawn on the
host in exactly the reference's stream order, mixture outcomes are picked on
the host (state independent, bit-exact), and a BATCH of trajectories runs
through the fused device passes; the outcome of each general site is chosen
on device from the reduced density matrix of its targets at the pass boundary
the planner opens for it (``ptsbe_run_conventional``,
``csrc/conventional.cuh``).  Shots then come from the same device sampler as
the PTSBE path: the trajectory's own PCG64 stream after its site draws
(per-trajectory path) or the ensemble stream's uniforms (dense path).
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from .errors import AnnihilatedStateError, ValidationError

# Circuits up to this width use the reference's dense-ensemble stream order in
# sample_conventional (trajectory.py:13-15); wider ones one PCG64 stream per trajectory.
DENSE_ENSEMBLE_LIMIT = 8
ANNIHILATED_MSG = "conventional draw annihilated a trajectory state"
KEY_SCALE = 9007199254740992.0   # 2^53: u = key * 2^-53 exactly


def select_index(r: float, probs) -> int:
    """Smallest k whose running sum of probs exceeds r; the last index if none does.

    The running sum is accumulated left to right in float64 -- the same
    rounding as ``np.cumsum`` -- so vectorised callers can use
    ``searchsorted(cumsum(probs), r, side="right")`` and stay bit-exact.
    """
    n = len(probs)
    if n == 0:
        raise ValidationError("empty probability list")
    running = 0.0
    for k, p in enumerate(probs):
        running += p
        if r < running:
            return k
    return n - 1


def select_indices(r: np.ndarray, probs) -> np.ndarray:
    """Vectorised ``select_index`` over an array of uniforms (bit-identical)."""
    edges = np.cumsum(np.asarray(probs, dtype=np.float64))
    k = np.searchsorted(edges, r, side="right")
    return np.minimum(k, len(edges) - 1)


@dataclass
class RealizedTrajectory:
    """One stochastic realization: a selection per site, in site firing order."""

    selections: list
    weight: float
    final_state: object    # statevector.ComplexState


class _Sites:
    """Firing order of the circuit's sites and the host half of each selection."""

    def __init__(self, circuit, prog):
        from .program import KIND_SITE
        self.fire = [so.ref for so in prog.stream if so.kind == KIND_SITE]
        self.S = prog.n_sites
        self.mix = []
        for sid in self.fire:
            ch = circuit.channels[circuit.site(sid).channel_id]
            m = ch.unitary_mixture()
            self.mix.append(None if m is None else np.asarray(m.probs, dtype=np.float64))
        self.any_general = any(m is None for m in self.mix)

    def tables(self, U: np.ndarray):
        """(T, S_fire) uniforms in firing order -> (sel by site id, uniforms by site id)."""
        T = U.shape[0]
        sel = np.zeros((T, self.S), dtype=np.uint8)
        ufull = np.zeros((T, self.S), dtype=np.float64)
        for j, sid in enumerate(self.fire):
            if self.mix[j] is not None:
                sel[:, sid] = select_indices(U[:, j], self.mix[j])
            else:
                ufull[:, sid] = U[:, j]
        return sel, ufull


def _engine_for(circuit, dtype: str, want: int):
    from .execute import get_engine
    return get_engine(circuit, dtype, want=want, conventional=True)


def _run_batch(eng, sites: _Sites, U: np.ndarray):
    """Device run of trajectories with site uniforms U (firing order): (sel, weights, status)."""
    sel, ufull = sites.tables(U)
    if sites.any_general:
        return eng.run_conventional(sel, ufull)
    w, st = eng.run(sel)
    return sel, w, st


def run_trajectory(circuit, rng: np.random.Generator, dtype: str = "c128") -> RealizedTrajectory:
    """Walk the ops; after each op fire its sites with one uniform draw per site (ref ``trajectory.py:40-70``).

    Unitary-mixture sites use the channel's fixed probabilities, general sites the
    branch probabilities ||K_k psi||^2 of the current state (computed on device)."""
    from .statevector import ComplexState
    eng = _engine_for(circuit, dtype, 1)
    sites = _Sites(circuit, eng.program)
    U = np.asarray(rng.random(len(sites.fire)), dtype=np.float64).reshape(1, -1)
    sel, w, st = _run_batch(eng, sites, U)
    if st[0] != 0:
        raise AnnihilatedStateError(f"Kraus selection annihilates the state (norm^2 = {w[0]:.3e})")
    amps = eng.get_state(0).astype(np.complex128, copy=False)
    selections = [(sid, int(sel[0, sid])) for sid in sites.fire]
    return RealizedTrajectory(selections, float(w[0]), ComplexState(circuit.n_qubits, amps))


def _mixture_joint_prob(circuit, selections):
    """Product of the mixture probabilities of every selection, None for a general channel
    (ref ``trajectory.py:128-136``; same multiplication order)."""
    p = 1.0
    for site_id, k in selections:
        mixture = circuit.channels[circuit.site(site_id).channel_id].unitary_mixture()
        if mixture is None:
            return None
        p *= float(mixture.probs[k])
    return p


def _conventional_row(circuit, t, selections, weight, counts, shots):
    return {
        "id": t,
        "selections": tuple((s, k) for s, k in selections if k != 0),
        "joint_prob": _mixture_joint_prob(circuit, selections),
        "realized_weight": weight,
        "shots": shots,
        "counts": counts,
        "seed": None,
        "status": "ok",
        "tags": {},
        "prep_time": None,
        "sample_time": None,
    }


def sample_conventional(circuit, n_traj: int, shots_per_traj: int = 1, master_seed: int = 0,
                        dtype: str = "c128"):
    """n_traj independent conventional trajectories, fresh state each, shots collected
    into a Dataset (ref ``trajectory.py:73-106``).

    Same random streams as the reference: for n <= DENSE_ENSEMBLE_LIMIT one
    PCG64(master_seed) consumed in (chunk, site)-major then (chunk, shot)-major
    order (``:138-219``), else PCG64(mix_seed(master_seed, t)) per trajectory (its
    site draws, then its shots).  Trajectories run in device batches.
    """
    from . import _native as N
    from .engine import pcg64_state_words
    from .execute import assemble_dataset, mix_seed

    if n_traj < 1:
        raise ValidationError(f"trajectory count must be >= 1, got {n_traj}")
    if shots_per_traj < 1:
        raise ValidationError(f"shots per trajectory must be >= 1, got {shots_per_traj}")
    start = time.perf_counter()
    n = circuit.n_qubits
    m = shots_per_traj
    dense = n <= DENSE_ENSEMBLE_LIMIT
    eng = _engine_for(circuit, dtype, n_traj)
    sites = _Sites(circuit, eng.program)
    S = len(sites.fire)
    fmt = f"0{n}b"
    rows = []

    def run_rows(t0, U, shot_arg):
        """Device batches over trajectories t0.. with site uniforms U; shot_arg(lo, hi) -> sample kwargs."""
        for lo in range(0, U.shape[0], eng.cap):
            hi = min(U.shape[0], lo + eng.cap)
            sel, w, st = _run_batch(eng, sites, U[lo:hi])
            if np.any(st != N.TRAJ_OK):
                raise AnnihilatedStateError(ANNIHILATED_MSG if dense else
                                            f"Kraus selection annihilates the state (norm^2 = {w[st != 0][0]:.3e})")
            out = eng.sample(np.full(hi - lo, m, dtype=np.int64), **shot_arg(lo, hi))
            for b in range(hi - lo):
                if dense:   # the ensemble records draws in site-id order (circuit.sites)
                    selections = [(s.site_id, int(sel[b, s.site_id])) for s in circuit.sites]
                else:
                    selections = [(sid, int(sel[b, sid])) for sid in sites.fire]
                a, z = int(out.offsets[b]), int(out.offsets[b + 1])
                counts = {format(int(v), fmt): int(c) for v, c in zip(out.indices[a:z], out.counts[a:z])}
                rows.append(_conventional_row(circuit, t0 + lo + b, selections, float(w[b]), counts, m))

    if dense:
        rng = np.random.Generator(np.random.PCG64(master_seed))
        chunk = int(min(65536, max(256, (1 << 21) // (1 << n))))
        done = 0
        while done < n_traj:
            b = min(chunk, n_traj - done)
            U = rng.random(S * b).reshape(S, b).T.copy()            # r = rng.random(b) per site
            keys = (rng.random(m * b).reshape(m, b).T * KEY_SCALE).astype(np.uint64)   # per shot j
            run_rows(done, U, lambda lo, hi, keys=keys: dict(rng_mode=N.RNG_KEYS, keys=keys[lo:hi].reshape(-1)))
            done += b
    else:
        U = np.empty((n_traj, S), dtype=np.float64)
        words = np.empty((n_traj, 4), dtype=np.uint64)
        for t in range(n_traj):
            g = np.random.Generator(np.random.PCG64(mix_seed(master_seed, t)))
            U[t] = g.random(S)
            words[t] = pcg64_state_words(g)       # the stream after the site draws: shots
        run_rows(0, U, lambda lo, hi: dict(rng_mode=N.RNG_PCG64, rng_state=words[lo:hi].reshape(-1)))
    wall = time.perf_counter() - start
    return assemble_dataset(circuit, rows, master_seed=master_seed, mode="conventional",
                            meta={"strategy": "conventional", "shots_per_trajectory": shots_per_traj},
                            wall_time=wall)
