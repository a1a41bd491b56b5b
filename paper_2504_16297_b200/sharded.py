"""Intra-trajectory state sharding for states too large for one GPU.

A state of ``n`` qubits is split over ``D = 2^k`` shards: shard ``s`` holds the
``2^(n-k)`` amplitudes whose top ``k`` physical bits equal ``s``.  Logical
qubits move between *local* bits (inside a shard) and *global* bits (the shard
index):

* the op stream (reference order, ``execute.py:85-97``) is cut into
  **segments** whose ops touch local qubits only; inside a segment every
  shard runs the same fused passes on its own amplitudes (the global bits are
  spectators), so a segment is just a pass range of an ordinary program
  compiled for ``n - k`` qubits (``ptsbe_run_range``);
* between segments the global qubits the next op needs are **swapped** with
  local ones (the local qubit used furthest in the future, Belady) -- all
  pairs due together in ONE all-to-all of 2^k' parts per shard group
  (``ptsbe_shard_swap``: grouped ``ncclSend``/``ncclRecv`` on a comm stream,
  chunked and double-buffered so part packing overlaps the NVLink transfer;
  ``ptsbe_shard_swap_local`` swaps parts in place between the shards of one
  process);
* renormalising (general) Kraus sites: the realized weight is a ratio of norms
  of the WHOLE state, so each shard reduces its slot norms and the sums are
  added over the shards -- ``ncclAllReduce`` on the engine stream inside
  ``ptsbe_run_range(PTSBE_SHARDED)``, or pass by pass through
  ``ptsbe_slot_norms`` / ``ptsbe_finalize_norms`` (one process, or a
  torch.distributed transport) -- so every shard applies the same weight and
  deferred renormalisation (ref ``statevector.py:136-145``, ``execute.py:93-97``);
* sampling: each shard's exact fixed-point CDF total (``ptsbe_norm_totals``,
  integers, so the split is exact) gives the multinomial split of the
  trajectory's shots over shards; every shard draws its share with its own
  Philox stream and the physical indices are mapped back to logical
  bitstrings.  (Bit-exact PCG64 replay needs the logical CDF order and is
  offered by the unsharded engine only.)

Transports: ``VirtualShards`` keeps all shards in one process (one device;
GPU tests and single-GPU validation up to 34 qubits), ``DistributedShards``
runs one shard per rank -- ``EngineShardBackend(transport="nccl")`` exchanges
through the engine's own NCCL communicator (the B200 path), ``"torch"``
through ``torch.distributed`` point-to-point ops (gloo in the CPU tests).
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np

from .errors import ValidationError
from .execute import mix_seed
from .program import Program, lower, plan_native, selection_matrix


@dataclass
class ShardPlan:
    n: int
    k: int
    segments: list                 # per segment: (pass_begin, pass_end)
    swaps: list                    # per segment: [(global bit g, local bit l)] applied AFTER it
    final_map: dict                # logical qubit -> ("L", bit) | ("G", bit)
    program: Program               # program over n - k local qubits
    initial_map: dict = field(default_factory=dict)
    pass_general: list = field(default_factory=list)   # per pass: has renormalising sites

    @property
    def n_local(self) -> int:
        return self.n - self.k

    @property
    def n_swaps(self) -> int:
        return sum(len(s) for s in self.swaps)

    @property
    def any_general(self) -> bool:
        return any(self.pass_general)


def _next_use(stream, start, q):
    for i in range(start, len(stream)):
        if q in stream[i].targets:
            return i
    return len(stream) + 1


def _segment_pass_counter(segments_ops, stream, nl, L, c):
    """Total passes of all segments under a local-bit relabelling sigma (native planner, no
    per-segment layout search): the objective of plan_sharded's layout search."""
    import ctypes as C

    from . import _native as N
    lib = N.load_library()
    segs = []
    for ops, mapping in segments_ops:
        if not ops:
            continue
        t0 = np.array([mapping[stream[i].targets[0]][1] for i in ops], dtype=np.int64)
        t1 = np.array([mapping[stream[i].targets[1]][1] if len(stream[i].targets) > 1 else -1 for i in ops],
                      dtype=np.int64)
        gen = np.array([(1 if stream[i].general else 0) | (2 if stream[i].kind == 0 else 0) for i in ops],
                       dtype=np.uint8)
        segs.append((t0, t1, gen))
    out_pass = np.zeros(max((len(t0) for t0, _, _ in segs), default=1) + 1, dtype=np.int32)
    out_masks = np.zeros(out_pass.size + 1, dtype=np.uint64)
    ptr = lambda a: C.c_void_p(a.ctypes.data)  # noqa: E731

    def count(sigma: np.ndarray) -> int:
        tot = 0
        for t0, t1, gen in segs:
            masks = (np.uint64(1) << sigma[t0].astype(np.uint64))
            has1 = t1 >= 0
            masks[has1] |= np.uint64(1) << sigma[t1[has1]].astype(np.uint64)
            perm = np.arange(nl, dtype=np.int32)
            P = lib.ptsbe_plan(nl, t0.size, ptr(masks), ptr(gen), L, c, 0, 0, ptr(perm), ptr(out_pass),
                               ptr(out_masks), out_masks.size)
            if P < 0:
                return 1 << 30
            tot += P
        return tot
    return count


def plan_sharded(circuit, k: int, dtype: str = "c64", tile_bits: int | None = None,
                 low_bits: int | None = None, search_iters: int | None = None, seed: int = 0) -> ShardPlan:
    """Segments of local-only ops with global<->local swaps between them.

    The segmentation (which ops run between which swaps) depends only on which qubits are
    global; the local BIT each local qubit occupies is free.  A local search over that
    labelling (random transpositions, sideways moves accepted -- the unsharded planner's
    layout search, with the summed pass count of every segment as its objective) cuts
    config 5's passes from 29 to about half."""
    from .program import DEFAULT_LOW_BITS, DEFAULT_TILE_BITS
    n = circuit.n_qubits
    if not 1 <= k < n - 2:
        raise ValidationError(f"cannot shard {n} qubits over 2^{k} shards")
    prog = lower(circuit)
    stream = prog.stream
    nl = n - k
    # initial layout: the k qubits used latest are global; local bits by usage (busiest lowest)
    first_use = {q: _next_use(stream, 0, q) for q in range(n)}
    glob = sorted(range(n), key=lambda q: (-first_use[q], q))[:k]
    uses = {q: sum(q in so.targets for so in stream) for q in range(n)}
    local = sorted((q for q in range(n) if q not in glob), key=lambda q: (-uses[q], q))
    where = {q: ("L", i) for i, q in enumerate(local)}
    where.update({q: ("G", i) for i, q in enumerate(glob)})
    initial = dict(where)
    segments_ops, swaps, cur = [], [], []
    for idx, so in enumerate(stream):
        need = [q for q in so.targets if where[q][0] == "G"]
        if need:
            segments_ops.append((cur, dict(where)))
            cur = []
            sw = []
            for q in need:
                cands = [r for r in range(n) if where[r][0] == "L" and r not in so.targets]
                victim = max(cands, key=lambda r: (_next_use(stream, idx, r), -r))
                g, l = where[q][1], where[victim][1]
                where[q], where[victim] = ("L", l), ("G", g)
                sw.append((g, l))
            swaps.append(sw)
        cur.append(idx)
    segments_ops.append((cur, dict(where)))
    swaps.append([])
    # one program over the local qubits: segments' passes back to back
    L = tile_bits if tile_bits is not None else DEFAULT_TILE_BITS[dtype]
    c = low_bits if low_bits is not None else DEFAULT_LOW_BITS[dtype]
    iters = (2000 if nl > L else 0) if search_iters is None else search_iters
    sigma = np.arange(nl, dtype=np.int64)           # local label -> physical local bit
    if iters > 0:
        count = _segment_pass_counter(segments_ops, stream, nl, min(L, nl), min(c, L, nl))
        best = count(sigma)
        rng = np.random.Generator(np.random.PCG64(seed))
        for _ in range(iters):
            a, b = rng.integers(0, nl, size=2)
            if a == b:
                continue
            cand = sigma.copy()
            cand[a], cand[b] = cand[b], cand[a]
            p = count(cand)
            if p <= best:
                best, sigma = p, cand
    relabel = lambda m: {q: (kind, int(sigma[bit]) if kind == "L" else bit) for q, (kind, bit) in m.items()}  # noqa: E731
    segments_ops = [(ops, relabel(mapping)) for ops, mapping in segments_ops]
    where = relabel(where)
    initial = relabel(initial)
    swaps = [[(g, int(sigma[l])) for g, l in sw] for sw in swaps]
    new_stream, passes, ranges = [], [], []
    for ops, mapping in segments_ops:
        seg_stream = [replace(stream[i], targets=tuple(mapping[q][1] for q in stream[i].targets)) for i in ops]
        base = len(new_stream)
        new_stream.extend(seg_stream)
        p0 = len(passes)
        if seg_stream:
            _, seg_passes = plan_native(nl, seg_stream, L, c, search_iters=0)
            for pp in seg_passes:
                pp.ops = [base + i for i in pp.ops]
            passes.extend(seg_passes)
        ranges.append((p0, len(passes)))
    sprog = Program(nl, new_stream, prog.mats, prog.chans, prog.chan_index, prog.site_chan,
                    passes=passes, g_ref=prog.g_ref, perm=None)
    pass_general = [any(new_stream[i].general for i in pp.ops) for pp in passes]
    return ShardPlan(n, k, ranges, swaps, dict(where), sprog, initial, pass_general)


def physical_to_logical(shard: np.ndarray, local_idx: np.ndarray, plan: ShardPlan) -> np.ndarray:
    """Logical basis index of (shard, local index) pairs under the final layout."""
    out = np.zeros(local_idx.shape, dtype=np.uint64)
    s = shard.astype(np.uint64)
    li = local_idx.astype(np.uint64)
    for q, (kind, bit) in plan.final_map.items():
        src = li if kind == "L" else s
        out |= ((src >> np.uint64(bit)) & np.uint64(1)) << np.uint64(q)
    return out


def _split_shots(totals: np.ndarray, m: int, seed: int) -> np.ndarray:
    """Multinomial split of m shots over shards with exact integer weights."""
    if m == 0:
        return np.zeros(totals.size, dtype=np.int64)
    t = totals.astype(np.float64)
    p = t / t.sum()
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.multinomial(m, p).astype(np.int64)


class VirtualShards:
    """All 2^k shards in one process on one device (GPU tests, single-GPU validation)."""

    def __init__(self, plan: ShardPlan, dtype: str = "c64", batch_cap: int = 1, device: int = 0):
        from .engine import Engine
        self.plan = plan
        self.dtype = dtype
        self.D = 1 << plan.k
        self.engines = [Engine(plan.n_local, dtype, batch_cap=batch_cap, device=device) for _ in range(self.D)]
        for e in self.engines:
            e.load_program(plan.program)

    def close(self):
        for e in self.engines:
            e.close()

    def run(self, sel: np.ndarray):
        """Prepare B trajectories over the shards; returns (weights, status) of the whole states."""
        from .engine import shard_swap_local
        B = sel.shape[0]
        plan = self.plan
        for i, (p0, p1) in enumerate(plan.segments):
            if plan.any_general:     # pass by pass: global norms of renormalising sites
                for p in range(p0, p1):
                    for s, e in enumerate(self.engines):
                        e.run_range(sel, p, p + 1, zero_vector=(p == 0 and s != 0),
                                    defer_norms=plan.pass_general[p])
                    if plan.pass_general[p]:
                        total = self.engines[0].slot_norms(B)
                        for e in self.engines[1:]:
                            total = total + e.slot_norms(B)      # fixed shard order
                        for e in self.engines:
                            e.finalize_norms(B, total)
            else:
                for s, e in enumerate(self.engines):   # only shard 0 holds |0...0> initially
                    e.run_range(sel, p0, p1, zero_vector=(p0 == 0 and s != 0))
            if plan.swaps[i]:
                shard_swap_local(self.engines, B, plan.swaps[i])
        return self.engines[0].get_weights(B)

    def sample(self, shots, seeds):
        """Philox shots per trajectory -> list of (logical indices sorted, counts)."""
        from . import _native as N
        shots = np.asarray(shots, dtype=np.int64)
        B = shots.size
        totals = np.stack([e.norm_totals(B) for e in self.engines], axis=1)   # (B, D)
        split = np.stack([_split_shots(totals[b], int(shots[b]), int(seeds[b])) for b in range(B)])
        per_traj = [[] for _ in range(B)]
        for s, e in enumerate(self.engines):
            keys = np.array([mix_seed(int(seeds[b]), s) for b in range(B)], dtype=np.uint64)
            out = e.sample(split[:, s], N.RNG_PHILOX, rng_state=keys)
            for b in range(B):
                lo, hi = out.offsets[b], out.offsets[b + 1]
                idx = physical_to_logical(np.full(hi - lo, s), out.indices[lo:hi], self.plan)
                per_traj[b].append((idx, out.counts[lo:hi]))
        result = []
        for b in range(B):
            idx = np.concatenate([x[0] for x in per_traj[b]]) if per_traj[b] else np.zeros(0, np.uint64)
            cnt = np.concatenate([x[1] for x in per_traj[b]]) if per_traj[b] else np.zeros(0, np.uint32)
            order = np.argsort(idx, kind="stable")
            result.append((idx[order], cnt[order]))
        return result

    def logical_state(self, b: int = 0) -> np.ndarray:
        """Assemble the full logical state of trajectory b (tests / small n)."""
        nl = self.plan.n_local
        parts = [e.get_state(b) for e in self.engines]
        phys_local = np.arange(1 << nl, dtype=np.uint64)
        out = np.zeros(1 << self.plan.n, dtype=parts[0].dtype)
        for s, amp in enumerate(parts):
            out[physical_to_logical(np.full(phys_local.size, s), phys_local, self.plan).astype(np.int64)] = amp
        return out


class DistributedShards:
    """One shard per rank (one process per GPU).

    ``backend`` is this rank's shard.  A backend with ``native = True`` (the engine's
    NCCL group, ``EngineShardBackend(transport="nccl")``) does swaps and cross-shard
    norms itself on the GPU; otherwise swaps go over ``torch.distributed`` P2P and the
    norms of renormalising sites through ``all_reduce`` pass by pass.
    """

    def __init__(self, plan: ShardPlan, backend, dtype: str = "c64", group=None):
        import torch.distributed as dist
        self.plan = plan
        self.dtype = dtype
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if self.world != 1 << plan.k:
            raise ValidationError(f"{self.world} ranks for 2^{plan.k} shards")
        self.backend = backend

    def run(self, sel: np.ndarray):
        """Prepare B trajectories; returns this rank's (weights, status) -- the same on every shard."""
        B = sel.shape[0]
        s = self.rank
        plan = self.plan
        native = getattr(self.backend, "native", False)
        for i, (p0, p1) in enumerate(plan.segments):
            if native or not plan.any_general:
                self.backend.run_range(sel, p0, p1, p0 == 0 and s != 0)
            else:
                for p in range(p0, p1):
                    self.backend.run_range(sel, p, p + 1, p == 0 and s != 0, defer_norms=plan.pass_general[p])
                    if plan.pass_general[p]:
                        self.backend.finalize_norms(B, self._all_reduce(self.backend.slot_norms(B)))
            if not plan.swaps[i]:
                continue
            if native:
                self.backend.swap(B, plan.swaps[i])      # one all-to-all for every pair due here
            else:
                for g, l in plan.swaps[i]:
                    self._swap_torch(B, g, l)
        return self.backend.get_weights(B)

    def _all_reduce(self, a: np.ndarray) -> np.ndarray:
        import torch
        import torch.distributed as dist
        t = torch.from_numpy(np.ascontiguousarray(a)).to(self.backend.comm_device())
        dist.all_reduce(t, group=self.group)
        return t.cpu().numpy()

    def _swap_torch(self, B, g, l):
        import torch.distributed as dist
        s = self.rank
        partner = s ^ (1 << g)
        v = 1 - ((s >> g) & 1)
        send = self.backend.half_buffer()
        recv = self.backend.half_buffer()
        for b in range(B):
            self.backend.exchange_half(b, l, v, send, unpack=False)
            self.backend.before_send()
            reqs = dist.batch_isend_irecv([dist.P2POp(dist.isend, send, partner, self.group),
                                           dist.P2POp(dist.irecv, recv, partner, self.group)])
            for r in reqs:
                r.wait()
            # NCCL's wait() only orders torch's current stream; the unpack runs on the
            # engine's own stream, so it must not start before the receive landed
            self.backend.after_recv()
            self.backend.exchange_half(b, l, v, recv, unpack=True)

    def sample(self, shots, seeds):
        """Returns per-trajectory (logical indices, counts) on rank 0, None elsewhere."""
        import torch
        import torch.distributed as dist
        shots = np.asarray(shots, dtype=np.int64)
        B = shots.size
        # collectives on the backend's device (an NCCL-only group cannot reduce CPU tensors)
        mine = torch.tensor(self.backend.norm_totals(B).astype(np.int64), device=self.backend.comm_device())
        allt = [torch.zeros_like(mine) for _ in range(self.world)]
        dist.all_gather(allt, mine, group=self.group)
        totals = np.stack([t.cpu().numpy().astype(np.uint64) for t in allt], axis=1)
        split = np.stack([_split_shots(totals[b], int(shots[b]), int(seeds[b])) for b in range(B)])
        keys = np.array([mix_seed(int(seeds[b]), self.rank) for b in range(B)], dtype=np.uint64)
        local = self.backend.sample(split[:, self.rank], keys)      # list of (local idx, counts)
        mapped = [(physical_to_logical(np.full(ix.size, self.rank), ix, self.plan), ct) for ix, ct in local]
        gathered = [None] * self.world if self.rank == 0 else None
        dist.gather_object(mapped, gathered, dst=dist.get_global_rank(self.group, 0) if self.group else 0,
                           group=self.group)
        if self.rank != 0:
            return None
        result = []
        for b in range(B):
            idx = np.concatenate([g[b][0] for g in gathered])
            cnt = np.concatenate([g[b][1] for g in gathered])
            order = np.argsort(idx, kind="stable")
            result.append((idx[order], cnt[order]))
        return result


def sharded_selection(plan: ShardPlan, specs) -> np.ndarray:
    return selection_matrix(plan.program, specs)


class EngineShardBackend:
    """This rank's shard on its GPU, for DistributedShards.

    ``transport="nccl"`` (default): the engine joins an NCCL group of the shard ranks
    (``ptsbe_shard_init``; rank 0 makes the id, ``group`` broadcasts it) and does the
    swaps and cross-shard norms on the GPU.  ``"torch"``: swaps over torch.distributed
    P2P with host-driven norms (any backend, e.g. gloo)."""

    def __init__(self, plan: ShardPlan, dtype: str = "c64", batch_cap: int = 1, device: int = 0,
                 transport: str = "nccl", group=None):
        from .engine import Engine, nccl_unique_id
        self.plan = plan
        self.dtype = dtype
        self.engine = Engine(plan.n_local, dtype, batch_cap=batch_cap, device=device)
        self.engine.load_program(plan.program)
        self.native = transport == "nccl"
        if self.native:
            import torch.distributed as dist
            rank, world = dist.get_rank(group), dist.get_world_size(group)
            obj = [nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group else 0, group=group)
            self.engine.shard_init(obj[0], rank, world)
        elif transport != "torch":
            raise ValidationError(f"unknown shard transport '{transport}'")

    def half_buffer(self):
        import torch
        cdt = torch.complex64 if self.dtype == "c64" else torch.complex128
        return torch.empty(1 << (self.plan.n_local - 1), dtype=cdt, device=torch.device("cuda", self.engine.device))

    def run_range(self, sel, p0, p1, zero_vector=False, defer_norms=False):
        self.engine.run_range(sel, p0, p1, zero_vector=zero_vector, defer_norms=defer_norms, sharded=self.native)

    def swap(self, B, pairs):
        self.engine.shard_swap(B, pairs)

    def slot_norms(self, B):
        return self.engine.slot_norms(B)

    def finalize_norms(self, B, sums):
        self.engine.finalize_norms(B, sums)

    def get_weights(self, B):
        return self.engine.get_weights(B)

    def comm_device(self):
        import torch
        return torch.device("cuda", self.engine.device)

    def before_send(self):
        # the pack ran on the engine's stream; torch's stream (NCCL's) must see it
        self.engine.synchronize()

    def after_recv(self):
        import torch
        torch.cuda.current_stream(self.comm_device()).synchronize()

    def exchange_half(self, b, bit, value, buf, unpack):
        self.engine.exchange_half(b, bit, value, buf.data_ptr(), unpack)

    def norm_totals(self, B):
        return self.engine.norm_totals(B)

    def sample(self, shots, keys):
        from . import _native as N
        out = self.engine.sample(shots, N.RNG_PHILOX, rng_state=keys)
        return [(out.indices[out.offsets[b]:out.offsets[b + 1]], out.counts[out.offsets[b]:out.offsets[b + 1]])
                for b in range(len(shots))]
