"""Python handle over one ``libptsbe.so`` engine (one device, one batch of states).

``Engine`` owns a device-resident batch of ``batch_cap`` statevectors of
2^n amplitudes (complex64 or complex128, qubit q = bit q of the index) and a
loaded program.  ``run`` prepares B trajectories at once from an outcome table
(the batched form of ``prepare_state``, reference ``execute.py:74-98``);
``sample`` draws every trajectory's shots in bulk (``sample_shots``,
``statevector.py:148-163``) and returns them run-length encoded.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import ValidationError
from .program import Program, compile_circuit

DTYPES = {"c64": (N.PTSBE_C64, np.complex64), "c128": (N.PTSBE_C128, np.complex128)}


def _ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data) if a is not None and a.size else None


def device_memory(device: int = 0):
    lib = N.load_library()
    free, total = C.c_uint64(), C.c_uint64()
    N.check(lib, None, lib.ptsbe_device_memory(device, C.byref(free), C.byref(total)), "device memory query")
    return int(free.value), int(total.value)


@dataclass
class Shots:
    """CSR shot output of one sample() call: trajectory b owns rows [offsets[b], offsets[b+1])."""

    indices: np.ndarray    # uint64 basis indices, ascending per trajectory
    counts: np.ndarray     # uint32
    offsets: np.ndarray    # int64, len B+1

    def counts_dict(self, b: int, n_qubits: int) -> dict:
        lo, hi = int(self.offsets[b]), int(self.offsets[b + 1])
        fmt = f"0{n_qubits}b"
        return {format(int(v), fmt): int(c) for v, c in zip(self.indices[lo:hi], self.counts[lo:hi])}


def program_args(prog: Program):
    """ptsbe_load_program arguments (after the handle), the physical layout, and the
    numpy buffers the pointer arguments refer to (keep them alive across the call)."""
    n = prog.n_qubits
    order = [(p, i) for p, plan in enumerate(prog.passes) for i in plan.ops]
    perm = list(range(n)) if prog.perm is None else list(prog.perm)
    ops = (N.Op * max(len(order), 1))()
    for j, (p, i) in enumerate(order):
        so = prog.stream[i]
        t0 = perm[so.targets[0]]
        t1 = perm[so.targets[1]] if len(so.targets) > 1 else -1
        ops[j] = N.Op(so.kind, len(so.targets), t0, t1, so.ref, p)
    mats = np.ascontiguousarray(np.ascontiguousarray(prog.mats.reshape(-1, 16)).view(np.float64).reshape(-1))
    chans = (N.Channel * max(len(prog.chans), 1))()
    for k, ch in enumerate(prog.chans):
        chans[k] = N.Channel(ch["n_outcomes"], ch["mat_base"], ch["general"], ch["arity"], ch["identity_mask"])
    site_chan = np.ascontiguousarray(prog.site_chan, dtype=np.int32)
    passes = (N.Pass * max(len(prog.passes), 1))()
    for p, plan in enumerate(prog.passes):
        passes[p] = N.Pass(plan.mask, len(plan.qubits), plan.low_bits)
    args = (ops, len(order), _ptr(mats), int(prog.mats.shape[0]), chans, len(prog.chans), _ptr(site_chan),
            int(site_chan.size), passes, len(prog.passes))
    return args, perm, (mats, site_chan)


def generated_source(prog: Program, dtype: str = "c64") -> str:
    """CUDA source of the circuit-specialised pass kernels for ``prog`` (host only, no GPU):
    the planner and code generator of ptsbe_load_program on a host-only handle."""
    lib = N.load_library()
    h = C.c_void_p()
    N.check(lib, None, lib.ptsbe_create_host(prog.n_qubits, DTYPES[dtype][0], C.byref(h)), "ptsbe_create_host")
    try:
        args, _, keep = program_args(prog)
        N.check(lib, h, lib.ptsbe_load_program(h, *args), "ptsbe_load_program (host only)")
        del keep
        n = lib.ptsbe_codegen_source(h, None, 0)
        buf = C.create_string_buffer(int(n) + 1)
        lib.ptsbe_codegen_source(h, buf, len(buf))
        return buf.value.decode()
    finally:
        lib.ptsbe_destroy(h)


class Engine:
    def __init__(self, n_qubits: int, dtype: str = "c128", batch_cap: int = 1, device: int = 0):
        if dtype not in DTYPES:
            raise ValidationError(f"dtype must be one of {sorted(DTYPES)}, got {dtype!r}")
        self.lib = N.load_library()
        self.n = int(n_qubits)
        self.dtype = dtype
        self.np_dtype = DTYPES[dtype][1]
        self.cap = int(batch_cap)
        self.device = int(device)
        self.program: Program | None = None
        h = C.c_void_p()
        st = self.lib.ptsbe_create(self.device, self.n, DTYPES[dtype][0], self.cap, C.byref(h))
        self.h = h
        if st != 0:
            msg = N.last_error(self.lib, h) if h.value else "invalid arguments"
            if h.value:
                self.lib.ptsbe_destroy(h)
            self.h = C.c_void_p()
            N.check(self.lib, None, st, f"ptsbe_create(n={n_qubits}, {dtype}, cap={batch_cap}): {msg}")

    # -- lifetime
    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.ptsbe_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _check(self, st, what):
        N.check(self.lib, self.h, st, what)

    # -- program
    def load(self, circuit, **plan_kw) -> Program:
        prog = compile_circuit(circuit, self.dtype, **plan_kw)
        self.load_program(prog)
        return prog

    def load_program(self, prog: Program) -> None:
        if prog.n_qubits != self.n:
            raise ValidationError(f"program is for {prog.n_qubits} qubits, engine holds {self.n}")
        args, perm, keep = program_args(prog)
        st = self.lib.ptsbe_load_program(self.h, *args)
        del keep
        self._check(st, "ptsbe_load_program")
        lay = np.array(perm, dtype=np.int32)
        self._check(self.lib.ptsbe_set_layout(self.h, C.c_void_p(lay.ctypes.data)), "ptsbe_set_layout")
        self.program = prog

    # -- execution
    def run(self, sel: np.ndarray, apply_only: bool = False):
        """Prepare len(sel) trajectories; returns (weights float64[B], status int32[B])."""
        sel = np.ascontiguousarray(sel, dtype=np.uint8)
        B = sel.shape[0]
        w = np.empty(B, dtype=np.float64)
        s = np.empty(B, dtype=np.int32)
        fn = self.lib.ptsbe_apply_program if apply_only else self.lib.ptsbe_run_batch
        self._check(fn(self.h, _ptr(sel), B, _ptr(w), _ptr(s), 0), "ptsbe_run_batch")
        return w, s

    def run_conventional(self, sel: np.ndarray, uniforms: np.ndarray, with_probs: bool = False):
        """Conventional trajectories (Algorithm 1, ref ``trajectory.py:40-70``): ``sel`` holds the
        unitary-mixture outcomes, general sites' outcomes are chosen on device from the state
        with ``uniforms[b, site]``.  Returns (final outcome table, weights, status[, probs])."""
        sel = np.ascontiguousarray(sel, dtype=np.uint8)
        B, S = sel.shape
        u = np.ascontiguousarray(uniforms, dtype=np.float64)
        if u.shape != (B, S):
            raise ValidationError(f"uniform table must be {(B, S)}, got {u.shape}")
        out = np.empty_like(sel)
        w = np.empty(B, dtype=np.float64)
        s = np.empty(B, dtype=np.int32)
        n_dec = sum(1 for so in self.program.stream if so.general) if self.program is not None else S
        probs = np.zeros((max(n_dec, 1), B, 64)) if with_probs else None
        self._check(self.lib.ptsbe_run_conventional(self.h, _ptr(sel), _ptr(u), B, _ptr(out), _ptr(w), _ptr(s),
                                                    _ptr(probs), 0), "ptsbe_run_conventional")
        return (out, w, s, probs) if with_probs else (out, w, s)

    def set_host_mirror(self, sel: np.ndarray | None, shots: np.ndarray | None) -> None:
        """Host copies of the device-resident inputs of the next ``mirror=True`` device calls
        (scheduling only: no device->host read-back per call).  Kept alive by the engine."""
        self._mirror = (None if sel is None else np.ascontiguousarray(sel, dtype=np.uint8),
                        None if shots is None else np.ascontiguousarray(shots, dtype=np.int64))
        a, b = self._mirror
        B = (a.shape[0] if a is not None else b.size) if (a is not None or b is not None) else 0
        self._check(self.lib.ptsbe_set_host_mirror(self.h, _ptr(a), _ptr(b), B), "ptsbe_set_host_mirror")

    def run_device(self, sel_ptr: int, B: int, w_ptr: int, s_ptr: int, sync: bool = False, mirror: bool = False):
        """Device-pointer variant (inputs already resident in HBM)."""
        flags = N.PTSBE_DEVICE_PTRS | (0 if sync else N.PTSBE_NO_SYNC) | (N.PTSBE_HOST_MIRROR if mirror else 0)
        self._check(self.lib.ptsbe_run_batch(self.h, C.c_void_p(sel_ptr), B, C.c_void_p(w_ptr),
                                             C.c_void_p(s_ptr), flags), "ptsbe_run_batch")

    def sample(self, shots, rng_mode: int = N.RNG_PCG64, rng_state=None, keys=None, out=None) -> Shots:
        """``out``: optional preallocated (indices uint64, counts uint32) host arrays with room for
        sum(shots) entries -- e.g. pinned memory, so the CSR read-back runs at full DMA speed."""
        shots = np.ascontiguousarray(shots, dtype=np.int64)
        B = shots.size
        total = int(shots.sum()) if B else 0
        if out is not None:
            idx, cnt = out
            if idx.dtype != np.uint64 or cnt.dtype != np.uint32 or idx.size < total or cnt.size < total \
                    or not (idx.flags.c_contiguous and cnt.flags.c_contiguous):
                raise ValidationError("sample output buffers: contiguous uint64 / uint32 with room for every shot")
        else:
            idx = np.empty(max(total, 1), dtype=np.uint64)
            cnt = np.empty(max(total, 1), dtype=np.uint32)
        nu = np.zeros(B, dtype=np.int64)
        rs = None if rng_state is None else np.ascontiguousarray(rng_state, dtype=np.uint64)
        ks = None if keys is None else np.ascontiguousarray(keys, dtype=np.uint64)
        st = self.lib.ptsbe_sample(self.h, B, _ptr(shots), rng_mode, _ptr(rs), _ptr(ks),
                                   _ptr(idx), _ptr(cnt), _ptr(nu), 0)
        self._check(st, "ptsbe_sample")
        off = np.zeros(B + 1, dtype=np.int64)
        np.cumsum(nu, out=off[1:])
        U = int(off[-1])
        return Shots(idx[:U], cnt[:U], off)

    def sample_device(self, B: int, shots_ptr: int, rng_mode: int, rng_ptr: int, idx_ptr: int, cnt_ptr: int,
                      nuniq_ptr: int, sync: bool = False, mirror: bool = False) -> None:
        """Device-pointer variant of sample(): inputs and CSR outputs stay in HBM."""
        flags = N.PTSBE_DEVICE_PTRS | (0 if sync else N.PTSBE_NO_SYNC) | (N.PTSBE_HOST_MIRROR if mirror else 0)
        st = self.lib.ptsbe_sample(self.h, B, C.c_void_p(shots_ptr), rng_mode, C.c_void_p(rng_ptr), None,
                                   C.c_void_p(idx_ptr), C.c_void_p(cnt_ptr), C.c_void_p(nuniq_ptr), flags)
        self._check(st, "ptsbe_sample")

    def gather(self, b: int, phys_idx) -> np.ndarray:
        """Normalised amplitudes of state b at PHYSICAL basis indices."""
        idx = np.ascontiguousarray(phys_idx, dtype=np.uint64)
        out = np.empty(idx.size, dtype=self.np_dtype)
        self._check(self.lib.ptsbe_gather_amplitudes(self.h, int(b), _ptr(idx), idx.size, _ptr(out)),
                    "ptsbe_gather_amplitudes")
        return out

    def get_state(self, b: int = 0) -> np.ndarray:
        out = np.empty(1 << self.n, dtype=self.np_dtype)
        self._check(self.lib.ptsbe_get_state(self.h, b, _ptr(out), 0), "ptsbe_get_state")
        return out

    def set_state(self, b: int, amps: np.ndarray) -> None:
        a = np.ascontiguousarray(amps, dtype=self.np_dtype)
        if a.size != 1 << self.n:
            raise ValidationError(f"state has {a.size} amplitudes, expected {1 << self.n}")
        self._check(self.lib.ptsbe_set_state(self.h, b, _ptr(a), 0), "ptsbe_set_state")

    def synchronize(self):
        self._check(self.lib.ptsbe_synchronize(self.h), "ptsbe_synchronize")

    @property
    def stream(self) -> int:
        return int(self.lib.ptsbe_stream(self.h) or 0)

    @property
    def launches(self) -> int:
        return int(self.lib.ptsbe_launch_count(self.h))

    def profile(self, enable: bool = True) -> None:
        self._check(self.lib.ptsbe_profile(self.h, 1 if enable else 0), "ptsbe_profile")

    def profile_read(self):
        """(pass-kernel ms, pass launches, algorithmic bytes) since profile(True)."""
        ms, n = C.c_double(), C.c_int64()
        self._check(self.lib.ptsbe_profile_read(self.h, C.byref(ms), C.byref(n)), "ptsbe_profile_read")
        return float(ms.value), int(n.value), float(self.lib.ptsbe_profile_bytes(self.h))

    def profile_passes(self):
        """Per pass index: (ms, algorithmic bytes) accumulated by profile_read()."""
        n = self.lib.ptsbe_profile_passes(self.h, None, None, 0)
        ms = np.zeros(max(n, 1))
        by = np.zeros(max(n, 1))
        self.lib.ptsbe_profile_passes(self.h, _ptr(ms), _ptr(by), n)
        return ms[:n], by[:n]

    def pass_info(self, p: int) -> dict:
        out = np.zeros(8, dtype=np.int64)
        self._check(self.lib.ptsbe_pass_info(self.h, int(p), _ptr(out), out.size), "ptsbe_pass_info")
        keys = ("L", "c", "gb", "n_phases", "n_ops", "n_slots", "threads", "codegen")
        return dict(zip(keys, (int(v) for v in out)))

    def info(self) -> dict:
        out = np.zeros(11, dtype=np.int64)
        self._check(self.lib.ptsbe_info(self.h, _ptr(out), out.size), "ptsbe_info")
        keys = ("n", "dtype", "cap", "n_passes", "tile_bits", "n_sites", "sample_bits", "norm_slots", "launches",
                "codegen", "n_phases")
        return dict(zip(keys, (int(v) for v in out)))


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id for ptsbe_shard_init (rank 0 makes it, the caller broadcasts it)."""
    lib = N.load_library()
    buf = C.create_string_buffer(128)
    N.check(lib, None, lib.ptsbe_nccl_unique_id(buf), "ptsbe_nccl_unique_id")
    return buf.raw


def shard_swap_local(engines, B: int, pairs) -> None:
    """Global<->local swap between the shards of one process (engines[s] holds shard s)."""
    lib = N.load_library()
    arr = (C.c_void_p * len(engines))(*[e.h.value for e in engines])
    g = np.array([p[0] for p in pairs], dtype=np.int32)
    lb = np.array([p[1] for p in pairs], dtype=np.int32)
    N.check(lib, engines[0].h, lib.ptsbe_shard_swap_local(arr, len(engines), int(B), len(pairs), _ptr(g), _ptr(lb)),
            "ptsbe_shard_swap_local")


def pcg64_state_words(seed_or_rng) -> np.ndarray:
    """(state_hi, state_lo, inc_hi, inc_lo) of a numpy PCG64 stream, for RNG_PCG64."""
    if isinstance(seed_or_rng, np.random.Generator):
        bg = seed_or_rng.bit_generator
    else:
        bg = np.random.PCG64(int(seed_or_rng))
    st = bg.state
    if st.get("bit_generator") != "PCG64":
        raise ValidationError("not a PCG64 stream")
    s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
    m = (1 << 64) - 1
    return np.array([s >> 64, s & m, inc >> 64, inc & m], dtype=np.uint64)


def _engine_sharding_methods():
    """Sharding primitives on Engine (ptsbe_run_range / exchange_half / norm_totals)."""

    def run_range(self, sel, pass_begin: int, pass_end: int, zero_vector: bool = False, continue_: bool = False,
                  defer_norms: bool = False, sharded: bool = False):
        """Passes [pass_begin, pass_end); from pass 0 the states start at |0...0> (or the zero
        vector) unless ``continue_``, which applies the range to the states as they are.
        ``defer_norms``: one pass of a shard whose renormalising norms are summed over the
        shards by the caller (slot_norms / finalize_norms); ``sharded``: a shard of an NCCL
        group (shard_init), norms all-reduced inside the engine."""
        sel = np.ascontiguousarray(sel, dtype=np.uint8)
        B = sel.shape[0]
        w = np.empty(B, dtype=np.float64)
        s = np.empty(B, dtype=np.int32)
        flags = (N.PTSBE_ZERO_VECTOR if zero_vector else 0) | (N.PTSBE_CONTINUE if continue_ else 0) | \
            (N.PTSBE_DEFER_NORMS if defer_norms else 0) | (N.PTSBE_SHARDED if sharded else 0)
        self._check(self.lib.ptsbe_run_range(self.h, _ptr(sel), B, int(pass_begin), int(pass_end), _ptr(w),
                                             _ptr(s), flags), "ptsbe_run_range")
        return w, s

    def exchange_half(self, b: int, bit: int, value: int, buf_ptr: int, unpack: bool):
        self._check(self.lib.ptsbe_exchange_half(self.h, int(b), int(bit), int(value), C.c_void_p(buf_ptr),
                                                 1 if unpack else 0), "ptsbe_exchange_half")

    def norm_totals(self, B: int) -> np.ndarray:
        out = np.zeros(B, dtype=np.uint64)
        self._check(self.lib.ptsbe_norm_totals(self.h, int(B), _ptr(out)), "ptsbe_norm_totals")
        return out

    def shard_init(self, nccl_id: bytes, rank: int, nranks: int):
        buf = C.create_string_buffer(bytes(nccl_id), 128)
        self._check(self.lib.ptsbe_shard_init(self.h, buf, int(rank), int(nranks)), "ptsbe_shard_init")

    def shard_swap(self, B: int, pairs):
        g = np.array([p[0] for p in pairs], dtype=np.int32)
        lb = np.array([p[1] for p in pairs], dtype=np.int32)
        self._check(self.lib.ptsbe_shard_swap(self.h, int(B), len(pairs), _ptr(g), _ptr(lb)), "ptsbe_shard_swap")

    def slot_norms(self, B: int) -> np.ndarray:
        """(slots, B) shard-local norm^2 of the pending pass's renormalising sites."""
        out = np.zeros((64, B), dtype=np.float64)
        n = C.c_int()
        self._check(self.lib.ptsbe_slot_norms(self.h, int(B), _ptr(out), C.byref(n)), "ptsbe_slot_norms")
        return out[: n.value].copy()

    def finalize_norms(self, B: int, sums: np.ndarray):
        a = np.ascontiguousarray(sums, dtype=np.float64)
        self._check(self.lib.ptsbe_finalize_norms(self.h, int(B), _ptr(a)), "ptsbe_finalize_norms")

    def get_weights(self, B: int):
        w = np.empty(B, dtype=np.float64)
        s = np.empty(B, dtype=np.int32)
        self._check(self.lib.ptsbe_get_weights(self.h, int(B), _ptr(w), _ptr(s)), "ptsbe_get_weights")
        return w, s

    Engine.run_range = run_range
    Engine.shard_init = shard_init
    Engine.shard_swap = shard_swap
    Engine.slot_norms = slot_norms
    Engine.finalize_norms = finalize_norms
    Engine.get_weights = get_weights
    Engine.exchange_half = exchange_half
    Engine.norm_totals = norm_totals


_engine_sharding_methods()
