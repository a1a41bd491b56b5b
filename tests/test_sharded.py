"""Intra-trajectory state sharding: planner invariants (CPU), a world-size-2 gloo run with a
CPU shard backend (test infrastructure), and virtual shards on the GPU vs the oracle."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import paper_2504_16297_b200 as P
from paper_2504_16297_b200 import workloads
from paper_2504_16297_b200.program import KIND_GATE
from paper_2504_16297_b200.sharded import (DistributedShards, ShardPlan, physical_to_logical, plan_sharded,
                                          sharded_selection)
from oracle import engine as O


def small_circuit(n=10, seed=3):
    text, noise = workloads.random_brickwork(n, layers=4, seed=seed, p=0.05)
    return P.attach_noise(P.parse_circuit(text), P.parse_noise_model(noise))


class NumpyShard:
    """CPU stand-in for one shard engine (oracle arithmetic) -- test infrastructure only.

    Mirrors the engine's sharded semantics: renormalising sites are applied unnormalised,
    their shard-local norms wait for the caller's cross-shard sums (slot_norms /
    finalize_norms), and the pass after a renormalising pass rescales by 1/sqrt(norm)."""

    native = False

    def __init__(self, plan: ShardPlan, B: int):
        self.plan = plan
        self.nl = plan.n_local
        self.states = [None] * B
        self.nst = np.ones(B)
        self.w = np.ones(B)
        self.prev_general = False
        self.pending = None

    def half_buffer(self):
        return torch.empty(1 << (self.nl - 1), dtype=torch.complex128)

    def comm_device(self):
        return torch.device("cpu")

    def before_send(self):
        pass

    def after_recv(self):
        pass

    def run_range(self, sel, p0, p1, zero_vector=False, defer_norms=False):
        prog = self.plan.program
        if p0 == 0:
            self.nst[:], self.w[:], self.prev_general = 1.0, 1.0, False
        for p in range(p0, p1):
            norms = []
            for b in range(sel.shape[0]):
                if p == 0:
                    self.states[b] = O.zero_state(self.nl)
                    if zero_vector:
                        self.states[b][0] = 0
                psi = self.states[b]
                if self.prev_general:
                    psi = psi / np.sqrt(self.nst[b])
                nb = []
                for i in prog.passes[p].ops:
                    so = prog.stream[i]
                    d = 1 << len(so.targets)
                    if so.kind == KIND_GATE:
                        m = prog.mats[so.ref][:d, :d]
                    else:
                        ch = prog.chans[int(prog.site_chan[so.ref])]
                        k = int(sel[b, so.ref])
                        if (ch["identity_mask"] >> k) & 1:
                            continue
                        m = prog.mats[ch["mat_base"] + k][:d, :d]
                    psi = O.apply_local(psi, m, so.targets, self.nl)
                    if so.kind != KIND_GATE and prog.chans[int(prog.site_chan[so.ref])]["general"]:
                        nb.append(float(np.sum(np.abs(psi) ** 2)))
                self.states[b] = psi
                norms.append(nb)
            self.prev_general = self.plan.pass_general[p]
            if self.prev_general:
                assert defer_norms and p1 == p + 1
                self.pending = np.array(norms, dtype=np.float64).T      # (slots, B)

    def slot_norms(self, B):
        return self.pending

    def finalize_norms(self, B, sums):
        for b in range(B):
            prev = 1.0
            for j in range(sums.shape[0]):
                self.w[b] *= sums[j, b] / prev
                prev = sums[j, b]
            self.nst[b] = prev
        self.pending = None

    def get_weights(self, B):
        return self.w[:B].copy(), np.zeros(B, dtype=np.int32)

    def _half_index(self, bit, value):
        i = np.arange(1 << (self.nl - 1))
        low = i & ((1 << bit) - 1)
        return ((i ^ low) << 1) | (value << bit) | low

    def exchange_half(self, b, bit, value, buf, unpack):
        idx = self._half_index(bit, value)
        if unpack:
            self.states[b][idx] = buf.numpy()
        else:
            buf.copy_(torch.from_numpy(self.states[b][idx].copy()))


def damped_circuit(n=10, seed=3):
    """Brickwork with amplitude damping (general channel) on ry and depolarizing on cx."""
    text, _ = workloads.random_brickwork(n, layers=3, seed=seed)
    return P.attach_noise(P.parse_circuit(text), P.parse_noise_model(
        "rule gate=ry qubit=* channel=amplitude_damping(0.1)\nrule gate=cx qubit=* channel=depolarizing(0.05)\n"))


def assemble(plan, shard_states):
    nl = plan.n_local
    loc = np.arange(1 << nl, dtype=np.uint64)
    out = np.zeros(1 << plan.n, dtype=np.complex128)
    for s, amp in enumerate(shard_states):
        out[physical_to_logical(np.full(loc.size, s), loc, plan).astype(np.int64)] = amp
    return out


@pytest.mark.parametrize("k", [1, 2])
def test_plan_invariants(k):
    c = small_circuit()
    plan = plan_sharded(c, k)
    prog = plan.program
    assert len(plan.segments) == len(plan.swaps) and plan.swaps[-1] == []
    assert sorted(q for q in plan.final_map) == list(range(c.n_qubits))
    assert sum(1 for v in plan.final_map.values() if v[0] == "G") == k
    for p in prog.passes:
        for i in p.ops:
            assert set(prog.stream[i].targets) <= set(p.qubits)
            assert max(prog.stream[i].targets) < plan.n_local
    assert len(prog.stream) == len(plan_sharded(c, k).program.stream)


def _worker(rank, world, port, q, damped):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = damped_circuit() if damped else small_circuit()
    plan = plan_sharded(c, 1)
    specs = P.presample_probabilistic(c, 50, 1, np.random.default_rng(4))[:3]
    shard = NumpyShard(plan, len(specs))
    w, st = DistributedShards(plan, shard).run(sharded_selection(plan, specs))
    gathered = [None] * world if rank == 0 else None
    states = [s / np.sqrt(shard.nst[b]) if shard.prev_general else s.copy() for b, s in enumerate(shard.states)]
    dist.gather_object((states, w.tolist()), gathered, dst=0)
    if rank == 0:
        q.put(([[g[0][b] for g in gathered] for b in range(len(specs))], [g[1] for g in gathered]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("damped", [False, True])
def test_world2_gloo_sharded_state_matches_oracle(damped):
    """Two ranks, one shard each: swaps over torch P2P, and with a general channel the
    norms of its sites all-reduced across the shards -> the oracle's state and weight."""
    c = damped_circuit() if damped else small_circuit()
    plan = plan_sharded(c, 1)
    assert plan.n_swaps >= 1
    assert plan.any_general == damped
    specs = P.presample_probabilistic(c, 50, 1, np.random.default_rng(4))[:3]
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    qq = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, qq, damped)) for r in range(2)]
    for p in procs:
        p.start()
    per_traj, weights = qq.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert weights[0] == weights[1]            # every shard holds the same weight
    for b, spec in enumerate(specs):
        ref, ref_w = O.prepare(c, spec.selections)
        got = assemble(plan, per_traj[b])
        assert np.linalg.norm(got - ref) <= 1e-12
        assert weights[0][b] == pytest.approx(ref_w, rel=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("k,dtype", [(1, "c128"), (2, "c128"), (2, "c64")])
def test_virtual_shards_match_oracle(k, dtype):
    from paper_2504_16297_b200.sharded import VirtualShards
    from paper_2504_16297_b200.execute import mix_seed
    from scipy import stats
    c = small_circuit(12, seed=5)
    plan = plan_sharded(c, k, dtype=dtype, tile_bits=6, low_bits=3)
    specs = P.presample_probabilistic(c, 60, 50_000, np.random.default_rng(6))[:3]
    vs = VirtualShards(plan, dtype, batch_cap=len(specs))
    try:
        vs.run(sharded_selection(plan, specs))
        tol = 1e-12 if dtype == "c128" else 1e-5
        for b, spec in enumerate(specs):
            ref, _ = O.prepare(c, spec.selections)
            got = vs.logical_state(b).astype(np.complex128)
            assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= tol
        seeds = [mix_seed(3, t) for t in range(len(specs))]
        res = vs.sample([s.shots for s in specs], seeds)
        for b, (idx, cnt) in enumerate(res):
            assert int(cnt.sum()) == specs[b].shots and np.all(np.diff(idx.astype(np.int64)) > 0)
            ref, _ = O.prepare(c, specs[b].selections)
            probs = np.abs(ref) ** 2
            assert np.all(probs[idx.astype(np.int64)] > 0)
            top = np.argsort(probs)[::-1][:10]
            obs = np.array([cnt[idx == t].sum() for t in top], dtype=float)
            exp = probs[top] * specs[b].shots
            obs = np.append(obs, specs[b].shots - obs.sum())
            exp = np.append(exp, specs[b].shots - exp.sum())
            assert stats.chisquare(obs, exp).pvalue > 1e-3   # the reference's chi^2 level (test_execute.py:168-178)
    finally:
        vs.close()


@pytest.mark.gpu
def test_virtual_shards_match_unsharded_engine_at_28_qubits():
    """sharded vs unsharded device runs at full size -- config 4 (28 q, c64) split
    into 2 shards of 27 local qubits (global<->local swaps between segments) must reproduce the
    unsharded engine's state for the same Kraus selections."""
    from paper_2504_16297_b200 import workloads
    from paper_2504_16297_b200.engine import Engine
    from paper_2504_16297_b200.program import selection_matrix
    from paper_2504_16297_b200.sharded import VirtualShards
    c = workloads.build(4, P.parse_circuit, P.parse_noise_model, P.attach_noise)
    specs = P.presample_probabilistic(c, 20, 100, np.random.default_rng(4))[1:2]
    plan = plan_sharded(c, 1, dtype="c64")
    assert plan.n_swaps >= 1
    vs = VirtualShards(plan, "c64", batch_cap=1)
    try:
        vs.run(sharded_selection(plan, specs))
        got = vs.logical_state(0).astype(np.complex128)
    finally:
        vs.close()
    with Engine(28, "c64", batch_cap=1) as eng:
        prog = eng.load(c)
        eng.run(selection_matrix(prog, specs))
        ref = eng.get_state(0).astype(np.complex128)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-5


def pair_swap_circuit(noise):
    """12 qubits whose last two qubits first meet in one cx: with k = 2 that op needs both
    global qubits at once -> one 2-pair all-to-all."""
    lines = ["qubits 12"] + [f"gate h {q}" for q in range(10)] + [f"gate cx {q} {q + 1}" for q in range(9)]
    lines += [f"gate ry {q} @ {0.3 + 0.1 * q}" for q in range(10)]
    lines += ["gate cx 10 11", "gate h 10", "gate cx 9 10", "gate cx 11 0", "gate ry 11 @ 0.7", "gate cx 4 11"]
    lines += [f"gate cx {q} {q + 1}" for q in range(0, 11, 2)]
    return P.attach_noise(P.parse_circuit("\n".join(lines) + "\n"), P.parse_noise_model(noise))


@pytest.mark.gpu
@pytest.mark.parametrize("k,dtype", [(1, "c128"), (2, "c128"), (3, "c128"), (2, "c64")])
def test_virtual_shards_general_channels_match_oracle(k, dtype):
    """Renormalising (amplitude-damping) sites sharded: slot norms summed over the shards,
    weights and states equal the oracle's (ref statevector.py:136-145, execute.py:93-97)."""
    from paper_2504_16297_b200.sharded import VirtualShards
    c = damped_circuit(12, seed=5)
    plan = plan_sharded(c, k, dtype=dtype, tile_bits=6, low_bits=3)
    assert plan.any_general and plan.n_swaps >= 1
    specs = P.presample_probabilistic(c, 60, 1, np.random.default_rng(6))[:4]
    tol = 1e-12 if dtype == "c128" else 1e-5
    vs = VirtualShards(plan, dtype, batch_cap=len(specs))
    try:
        w, st = vs.run(sharded_selection(plan, specs))
        for b, spec in enumerate(specs):
            try:
                ref, ref_w = O.prepare(c, spec.selections)
            except O.Annihilated:
                assert st[b] == 2
                continue
            assert st[b] == 0
            assert w[b] == pytest.approx(ref_w, rel=tol)
            got = vs.logical_state(b).astype(np.complex128)
            assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= tol
            for e in vs.engines[1:]:      # every shard carries the same weight
                assert e.get_weights(len(specs))[0][b] == w[b]
    finally:
        vs.close()


@pytest.mark.gpu
@pytest.mark.parametrize("noise", ["rule gate=* qubit=* channel=depolarizing(0.05)\n",
                                   "rule gate=ry qubit=* channel=amplitude_damping(0.2)\n"])
def test_virtual_shards_two_pair_all_to_all(noise):
    """An op on two global qubits: both pairs swapped in ONE 2^2-part all-to-all."""
    from paper_2504_16297_b200.sharded import VirtualShards
    c = pair_swap_circuit(noise)
    plan = plan_sharded(c, 2, dtype="c128", tile_bits=6, low_bits=3)
    assert max(len(sw) for sw in plan.swaps) == 2
    specs = P.presample_probabilistic(c, 60, 1, np.random.default_rng(2))[:3]
    vs = VirtualShards(plan, "c128", batch_cap=len(specs))
    try:
        w, st = vs.run(sharded_selection(plan, specs))
        for b, spec in enumerate(specs):
            ref, ref_w = O.prepare(c, spec.selections)
            got = vs.logical_state(b)
            assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-12
            assert w[b] == pytest.approx(ref_w, rel=1e-12)
    finally:
        vs.close()


@pytest.mark.gpu
def test_nccl_shard_group_single_rank(monkeypatch):
    """The engine's own NCCL path on one GPU: a 1-rank shard group.  (a) PTSBE_SHARDED runs
    all-reduce the renormalising norms inside the engine (identity over one rank) and give the
    unsharded weights/state; (b) the chunked grouped send/recv pipeline of ptsbe_shard_swap with
    every part addressed to the rank itself returns the state unchanged, bit for bit."""
    from paper_2504_16297_b200.engine import Engine, nccl_unique_id
    from paper_2504_16297_b200.program import compile_circuit, selection_matrix
    c = damped_circuit(12, seed=5)
    prog = compile_circuit(c, "c128", tile_bits=6, low_bits=3, search_iters=0)   # shard layouts are unpermuted
    specs = P.presample_probabilistic(c, 60, 1, np.random.default_rng(6))[:3]
    sel = selection_matrix(prog, specs)
    with Engine(12, "c128", batch_cap=3) as ref_eng, Engine(12, "c128", batch_cap=3) as eng:
        ref_eng.load_program(prog)
        w0, s0 = ref_eng.run(sel)
        eng.load_program(prog)
        eng.shard_init(nccl_unique_id(), 0, 1)
        w1, s1 = eng.run_range(sel, 0, prog.n_passes, sharded=True)
        assert np.array_equal(s0, s1)
        np.testing.assert_allclose(w1, w0, rtol=1e-13)
        for b in range(3):
            a, r = eng.get_state(b), ref_eng.get_state(b)
            assert np.linalg.norm(a - r) <= 1e-13 * np.linalg.norm(r)
        before = [eng.get_state(b) for b in range(3)]
        monkeypatch.setenv("PTSBE_SHARD_SELF_TEST", "1")
        monkeypatch.setenv("PTSBE_SHARD_CHUNK", "100")       # many chunks: exercises the double buffering
        eng.shard_swap(3, [(0, 4), (1, 7)])
        for b in range(3):
            assert np.array_equal(eng.get_state(b), before[b])
