"""Single-state API of the reference engine, executed by the CUDA engine.

Mirror of ``pkg/src/trajsim/statevector.py`` (the "inner engine boundary" of
SURVEY section 8b): ``ComplexState`` / ``ShotBatch`` keep the reference's host
representation (numpy amplitudes, qubit q = bit q; counts keyed by bitstrings
with qubit n-1 leftmost), while every transformation and every shot runs on
the device through ``libptsbe.so``.  Calls are functional -- inputs are never
mutated (ref ``statevector.py:121,145``).  These per-op entry points upload
and download the state each call, exactly like the reference allocates a new
array per op; the batched path (``execute.py``) keeps states resident.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .engine import Engine, pcg64_state_words
from .errors import AnnihilatedStateError, ValidationError
from .program import compile_ops

# Device states are not capped at the reference's 24 qubits; 30 bounds the
# host-side numpy copy these per-op calls round-trip (16 GiB at complex128).
MAX_QUBITS = 30
NORM_TOL = 1e-10
ANNIHILATION_TOL = 1e-14
DEFAULT_DTYPE = "c128"


@dataclass
class ComplexState:
    """Amplitude vector of a pure n-qubit state; bit q of a basis index is qubit q."""

    n_qubits: int
    amplitudes: np.ndarray

    def norm(self) -> float:
        return float(np.linalg.norm(self.amplitudes))

    def probabilities(self) -> np.ndarray:
        return np.abs(self.amplitudes) ** 2

    def copy(self) -> "ComplexState":
        return ComplexState(self.n_qubits, self.amplitudes.copy())


@dataclass
class ShotBatch:
    """bitstring -> multiplicity, qubit n-1 leftmost (ref ``statevector.py:35-61``)."""

    n_qubits: int
    counts: dict
    total: int

    @classmethod
    def from_indices(cls, indices: np.ndarray, n_qubits: int) -> "ShotBatch":
        vals, reps = np.unique(np.asarray(indices), return_counts=True)
        fmt = f"0{n_qubits}b"
        return cls(n_qubits, {format(int(v), fmt): int(c) for v, c in zip(vals, reps)}, int(np.size(indices)))

    @classmethod
    def from_runs(cls, indices: np.ndarray, counts: np.ndarray, n_qubits: int) -> "ShotBatch":
        fmt = f"0{n_qubits}b"
        d = {format(int(v), fmt): int(c) for v, c in zip(indices, counts)}
        return cls(n_qubits, d, int(np.sum(counts, dtype=np.int64)))

    def bitstrings(self):
        for bits in sorted(self.counts):
            for _ in range(self.counts[bits]):
                yield bits

    def merged(self, other: "ShotBatch") -> "ShotBatch":
        if other.n_qubits != self.n_qubits:
            raise ValidationError("cannot merge shot batches of different widths")
        out = dict(self.counts)
        for bits, c in other.counts.items():
            out[bits] = out.get(bits, 0) + c
        return ShotBatch(self.n_qubits, out, self.total + other.total)


_pool_lock = threading.Lock()
_pool: dict = {}


def _engine(n: int, dtype: str = DEFAULT_DTYPE) -> Engine:
    """Per-thread single-state engine (handles are not shared across threads)."""
    key = (threading.get_ident(), n, dtype)
    with _pool_lock:
        eng = _pool.get(key)
        if eng is None:
            eng = Engine(n, dtype, batch_cap=1)
            _pool[key] = eng
    return eng


def init_zero(n: int) -> ComplexState:
    if not 1 <= n <= MAX_QUBITS:
        raise ValidationError(f"qubit count must be in [1, {MAX_QUBITS}], got {n}")
    amps = np.zeros(1 << n, dtype=np.complex128)
    amps[0] = 1.0
    return ComplexState(n, amps)


def _check_targets(n: int, targets, dim: int) -> None:
    k = len(targets)
    if dim != 1 << k:
        raise ValidationError(f"matrix dimension {dim} does not fit {k} target qubit(s)")
    if len(set(targets)) != k:
        raise ValidationError(f"duplicate target in {tuple(targets)}")
    for t in targets:
        if not 0 <= t < n:
            raise ValidationError(f"target qubit {t} out of range for {n} qubits")


def _run_single(state: ComplexState, matrix, targets, general: bool):
    eng = _engine(state.n_qubits)
    prog = compile_ops(state.n_qubits, [(np.asarray(matrix, dtype=np.complex128), targets, general)], eng.dtype)
    eng.load_program(prog)
    eng.set_state(0, state.amplitudes)
    w, st = eng.run(np.zeros((1, prog.n_sites), dtype=np.uint8), apply_only=True)
    return eng, float(w[0]), int(st[0])


def apply_matrix(state: ComplexState, matrix: np.ndarray, targets) -> ComplexState:
    matrix = np.asarray(matrix)
    _check_targets(state.n_qubits, targets, matrix.shape[0])
    eng, _w, _s = _run_single(state, matrix, targets, general=False)
    return ComplexState(state.n_qubits, eng.get_state(0).astype(np.complex128, copy=False))


def apply_gate(state: ComplexState, op) -> ComplexState:
    return apply_matrix(state, op.matrix, op.targets)


def kraus_outcome_probability(state: ComplexState, kraus: np.ndarray, targets) -> float:
    """||K psi||^2 without changing the state (ref ``statevector.py:129-133``)."""
    kraus = np.asarray(kraus)
    _check_targets(state.n_qubits, targets, kraus.shape[0])
    _eng, w, _st = _run_single(state, kraus, targets, general=True)
    return w   # reported for annihilating outcomes too (the reference returns the raw norm^2)


def apply_kraus_normalized(state: ComplexState, kraus: np.ndarray, targets):
    """psi -> K psi / ||K psi|| and realized ||K psi||^2 (ref ``statevector.py:136-145``)."""
    kraus = np.asarray(kraus)
    _check_targets(state.n_qubits, targets, kraus.shape[0])
    eng, w, st = _run_single(state, kraus, targets, general=True)
    if st == N.TRAJ_ANNIHILATED:
        raise AnnihilatedStateError(f"Kraus selection annihilates the state (norm^2 = {w:.3e})")
    return ComplexState(state.n_qubits, eng.get_state(0).astype(np.complex128, copy=False)), w


def rng_words(rng: np.random.Generator):
    """(mode, words) for drawing from ``rng`` on the device, or None if not PCG64."""
    try:
        return pcg64_state_words(rng)
    except ValidationError:
        return None


def sample_shots(state: ComplexState, m: int, rng: np.random.Generator) -> ShotBatch:
    """m shots from |psi|^2 consuming exactly m uniforms of ``rng`` (ref ``statevector.py:148-163``).

    A PCG64 generator is replayed on the device (bit-exact uniforms) and then
    advanced by m on the host; any other generator supplies its m uniforms as
    53-bit keys.
    """
    if m < 1:
        raise ValidationError(f"shot count must be >= 1, got {m}")
    total = float(np.sum(np.abs(state.amplitudes) ** 2))
    if abs(total - 1.0) > 1e-6:
        raise ValidationError(f"state norm^2 = {total}, too far from 1 to sample")
    eng = _engine(state.n_qubits)
    eng.set_state(0, state.amplitudes)
    words = rng_words(rng)
    shots = np.array([m], dtype=np.int64)
    if words is not None:
        out = eng.sample(shots, N.RNG_PCG64, rng_state=words)
        rng.bit_generator.advance(m)
    else:
        keys = (rng.random(m) * 9007199254740992.0).astype(np.uint64)
        out = eng.sample(shots, N.RNG_KEYS, keys=keys)
    return ShotBatch.from_runs(out.indices, out.counts, state.n_qubits)
