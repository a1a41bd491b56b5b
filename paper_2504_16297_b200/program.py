"""Host compiler: NoisyCircuit -> device program (op stream, operator table, fused passes).

The reference evolves a trajectory by walking ``circuit.ops`` and, after each
gate, firing that gate's noise sites in site-id order with outcome
``chosen.get(site, 0)`` (``execute.py:85-97``) -- one full numpy pass per op
and per site.  This module lowers the same sequence once per circuit:

* a linear op stream: gate, then its sites (site-id order); a site op carries
  the site id and its channel, the outcome is read per trajectory on device;
* an operator table (complex128, 4x4 padded): gate matrices, unitary-mixture
  ``U_k`` (``noise.py:100-119``) or general ``K_k`` per channel outcome, with a
  mask of outcomes that are exactly the identity (skipped on device -- the
  builtin mixtures' ``U_0`` is exactly I, so the skip is bit-exact);
* a fusion plan: a partition of the stream into passes.  Each pass owns a
  tile qubit set Q (|Q| = L, always containing qubits 0..c-1 so tile rows are
  >= 128 B contiguous) and takes every op whose targets lie in Q and whose
  predecessors on those qubits already ran.  A pass is one HBM read + write
  of every state in the batch, regardless of how many ops it absorbs.

Planner: greedy in stream order.  Ops whose targets fit in the growing set
join; an op that does not fit blocks its qubits for the rest of the pass
(later ops on them depend on it), ops on untouched qubits keep flowing.
Sites of general (renormalising) channels never overtake one another: their
realized weights are ratios of consecutive norms in the reference's order
(statevector.py:136-145), so that order is part of the semantics.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import ValidationError

KIND_GATE = 0
KIND_SITE = 1

# 32-KB tiles for complex64; 64-KB single-buffered tiles for complex128 (config 4: 12 passes
# instead of 17 at 11 bits -- 566 K vs 473 K shots/s on one B200).
# complex128 tiles are made of 512-B rows (5 contiguous low qubits): fewer, longer DRAM
# bursts per tile, and the layout search still finds 11 passes for config 4 (882 K vs
# 831 K shots/s with 128-B rows; complex64 keeps 128-B rows: 1.81 M at 256-B vs 1.83 M).
DEFAULT_TILE_BITS = {"c64": 12, "c128": 12}
DEFAULT_LOW_BITS = {"c64": 4, "c128": 5}     # rows of 16 x 8 B = 128 B (c64) / 32 x 16 B = 512 B (c128)


@dataclass
class StreamOp:
    kind: int
    targets: tuple
    ref: int              # gate: matrix index; site: site id
    pos: int              # op position in circuit.ops
    general: bool = False # site of a non-unitary channel (renormalising)


@dataclass
class PassPlan:
    qubits: tuple         # sorted tile qubit set
    low_bits: int         # contiguous run 0..c-1 inside qubits
    ops: list             # stream indices, execution order

    @property
    def mask(self) -> int:
        m = 0
        for q in self.qubits:
            m |= 1 << q
        return m


@dataclass
class Program:
    n_qubits: int
    stream: list
    mats: np.ndarray              # (n_mats, 4, 4) complex128
    chans: list                   # dicts: n_outcomes, mat_base, general, arity, identity_mask
    chan_index: dict              # channel_id -> channel row
    site_chan: np.ndarray         # (S,) int32
    passes: list = field(default_factory=list)
    g_ref: int = 0                # reference-equivalent full-state passes: #ops + #sites
    perm: list = None             # logical qubit -> physical bit (None = identity)
    decide_general: bool = False  # planned for conventional trajectories (general sites open passes)

    @property
    def n_sites(self) -> int:
        return int(self.site_chan.size)

    @property
    def n_passes(self) -> int:
        return len(self.passes)


class _MatTable:
    def __init__(self):
        self.rows = []
        self.index = {}

    def add(self, m: np.ndarray, dedupe: bool = True) -> int:
        m = np.asarray(m, dtype=np.complex128)
        d = m.shape[0]
        pad = np.zeros((4, 4), dtype=np.complex128)
        pad[:d, :d] = m
        key = (d, pad.tobytes())
        if dedupe and key in self.index:
            return self.index[key]
        self.rows.append(pad)
        self.index[key] = len(self.rows) - 1
        return len(self.rows) - 1


def _is_identity(m: np.ndarray) -> bool:
    return bool(np.array_equal(m, np.eye(m.shape[0], dtype=np.complex128)))


def lower(circuit) -> Program:
    """Op stream + operator table of a circuit (no fusion yet)."""
    table = _MatTable()
    chans, chan_index = [], {}
    for cid, ch in circuit.channels.items():
        if ch.arity > 2:
            raise ValidationError(f"channel '{cid}': arity {ch.arity} unsupported on device (1 or 2)")
        mix = ch.unitary_mixture()
        ops = list(mix.unitaries) if mix is not None else list(ch.kraus_ops)
        if len(ops) > 64:
            raise ValidationError(f"channel '{cid}' has {len(ops)} outcomes (device limit 64)")
        base = len(table.rows)
        ident = 0
        for k, m in enumerate(ops):
            table.add(m, dedupe=False)
            if mix is not None and _is_identity(m):
                ident |= 1 << k
        chan_index[cid] = len(chans)
        chans.append(dict(n_outcomes=len(ops), mat_base=base, general=int(mix is None),
                          arity=ch.arity, identity_mask=ident))
    site_chan = np.array([chan_index[s.channel_id] for s in circuit.sites], dtype=np.int32)
    by_pos = circuit.sites_by_position()
    stream = []
    for pos, op in enumerate(circuit.ops):
        k = len(op.targets)
        if k > 2:
            raise ValidationError(f"op {pos} ('{op.name}') acts on {k} qubits; the device engine supports 1 or 2")
        if not _is_identity(op.matrix):
            stream.append(StreamOp(KIND_GATE, tuple(op.targets), table.add(op.matrix), pos))
        for s in by_pos.get(pos, ()):
            general = bool(chans[chan_index[s.channel_id]]["general"])
            stream.append(StreamOp(KIND_SITE, tuple(s.targets), s.site_id, pos, general))
    mats = np.array(table.rows, dtype=np.complex128).reshape(-1, 4, 4)
    return Program(circuit.n_qubits, stream, mats, chans, chan_index, site_chan,
                   g_ref=len(circuit.ops) + len(circuit.sites))


def plan_passes(n: int, stream: list, tile_bits: int, low_bits: int) -> list:
    """Greedy qubit-set fusion of the op stream into passes (see module docstring)."""
    L = min(n, tile_bits)
    if n <= L:
        return [PassPlan(tuple(range(n)), n, list(range(len(stream))))] if stream else []
    c = min(low_bits, L)
    low = frozenset(range(c))
    remaining = list(range(len(stream)))
    plans = []
    while remaining:
        qset = set(low)
        blocked = set()
        gen_blocked = False
        taken, deferred = [], []
        for i in remaining:
            so = stream[i]
            t = so.targets
            if blocked.intersection(t) or (so.general and gen_blocked):
                deferred.append(i)
                blocked.update(t)
                gen_blocked = gen_blocked or so.general
                continue
            grown = qset.union(t)
            if len(grown) <= L:
                qset = grown
                taken.append(i)
            else:
                deferred.append(i)
                blocked.update(t)
                gen_blocked = gen_blocked or so.general
        if not taken:     # cannot happen for arity <= 2 and L >= c + 2
            raise ValidationError("fusion planner made no progress")
        # pad the set with the lowest free qubits: longer contiguous rows, same traffic
        q = 0
        while len(qset) < L:
            if q not in qset:
                qset.add(q)
            q += 1
        qs = tuple(sorted(qset))
        run = 0
        while run < len(qs) and qs[run] == run:
            run += 1
        plans.append(PassPlan(qs, run, taken))
        remaining = deferred
    return plans


def plan_native(n: int, stream: list, tile_bits: int, low_bits: int, search_iters: int = 0,
                seed: int = 0, perm=None, decide_general: bool = False):
    """Same greedy rule in libptsbe (planner.h) plus a local search over the
    physical qubit layout; returns (perm logical->physical, passes in physical qubits).

    ``decide_general``: every general-channel site opens its pass, so its outcome
    can be chosen on device from the state at the pass boundary (conventional
    trajectories, ``ptsbe_run_conventional``)."""
    import ctypes as C

    from . import _native as N
    lib = N.load_library()
    m = len(stream)
    masks = np.zeros(max(m, 1), dtype=np.uint64)
    general = np.zeros(max(m, 1), dtype=np.uint8)
    for i, so in enumerate(stream):
        for q in so.targets:
            masks[i] |= np.uint64(1 << q)
        general[i] = (1 if so.general else 0) | (2 if so.kind == KIND_GATE else 0) | \
            (4 if (decide_general and so.general) else 0)
    p = np.arange(n, dtype=np.int32) if perm is None else np.array(perm, dtype=np.int32)
    out_pass = np.zeros(max(m, 1), dtype=np.int32)
    out_masks = np.zeros(max(m, 1) + 1, dtype=np.uint64)
    ptr = lambda a: C.c_void_p(a.ctypes.data)  # noqa: E731
    P = lib.ptsbe_plan(n, m, ptr(masks), ptr(general), tile_bits, low_bits, search_iters, seed,
                       ptr(p), ptr(out_pass), ptr(out_masks), out_masks.size)
    if P < 0:
        raise ValidationError("fusion planner failed")
    plans = []
    for k in range(P):
        mask = int(out_masks[k])
        qs = tuple(q for q in range(n) if (mask >> q) & 1)
        run = 0
        while run < len(qs) and qs[run] == run:
            run += 1
        plans.append(PassPlan(qs, run, [i for i in range(m) if out_pass[i] == k]))
    return [int(x) for x in p], plans


def default_search_iters(n: int, tile_bits: int) -> int:
    return 3000 if n > tile_bits else 0


def compile_circuit(circuit, dtype: str = "c128", tile_bits: int | None = None,
                    low_bits: int | None = None, search_iters: int | None = None, seed: int = 0,
                    decide_general: bool = False) -> Program:
    """Lower + plan.  Circuits wider than a tile get a physical qubit layout chosen
    by local search to minimise HBM passes (shots and states stay logical).
    ``decide_general`` plans for conventional trajectories (see ``plan_native``)."""
    prog = lower(circuit)
    L = tile_bits if tile_bits is not None else DEFAULT_TILE_BITS[dtype]
    c = low_bits if low_bits is not None else DEFAULT_LOW_BITS[dtype]
    n = circuit.n_qubits
    iters = default_search_iters(n, L) if search_iters is None else search_iters
    prog.perm, prog.passes = plan_native(n, prog.stream, L, c, iters, seed, decide_general=decide_general)
    prog.decide_general = decide_general
    return prog


def compile_ops(n: int, items, dtype: str = "c128") -> Program:
    """Program for an explicit list of (matrix, targets, general) ops -- the inner API.

    Each general op becomes a one-outcome general channel site, so the engine
    reports its realized norm^2 through the weight (statevector.py:129-145).
    """
    table = _MatTable()
    chans, stream, site_chan = [], [], []
    for matrix, targets, general in items:
        targets = tuple(int(t) for t in targets)
        if len(targets) > 2:
            raise ValidationError(f"{len(targets)}-qubit operators are unsupported on device (1 or 2)")
        if general:
            base = table.add(matrix, dedupe=False)
            chans.append(dict(n_outcomes=1, mat_base=base, general=1, arity=len(targets), identity_mask=0))
            sid = len(site_chan)
            site_chan.append(len(chans) - 1)
            stream.append(StreamOp(KIND_SITE, targets, sid, 0, True))
        else:
            stream.append(StreamOp(KIND_GATE, targets, table.add(matrix), 0))
    mats = np.array(table.rows, dtype=np.complex128).reshape(-1, 4, 4)
    prog = Program(n, stream, mats, chans, {}, np.array(site_chan, dtype=np.int32), g_ref=len(stream))
    prog.passes = plan_passes(n, stream, DEFAULT_TILE_BITS[dtype], DEFAULT_LOW_BITS[dtype])
    return prog


def selection_matrix(program: Program, specs) -> np.ndarray:
    """(B, S) uint8 outcome table: sel[b, site] = k for spec b's (site, k) pairs, else 0."""
    sel = np.zeros((len(specs), max(program.n_sites, 0)), dtype=np.uint8)
    for b, spec in enumerate(specs):
        for sid, k in spec.selections:
            sel[b, sid] = k
    return sel


def site_passes(program: Program) -> np.ndarray:
    """Pass index of every site of a planned program (-1: not in any pass)."""
    sp = np.full(program.n_sites, -1, dtype=np.int64)
    for p, plan in enumerate(program.passes):
        for i in plan.ops:
            so = program.stream[i]
            if so.kind == KIND_SITE:
                sp[so.ref] = p
    return sp


def prefix_order(program: Program, specs) -> list:
    """Execution order that puts trajectories with common outcome prefixes (in pass order) next
    to each other: batches of neighbours share more of the engine's tree schedule (a group of
    trajectories with identical outcomes through pass k is computed once through pass k)."""
    sp = site_passes(program)
    keys = [tuple(sorted((int(sp[sid]), sid, k) for sid, k in spec.selections)) for spec in specs]
    return sorted(range(len(specs)), key=lambda i: (keys[i], i))
