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
    """CPU stand-in for one shard engine (oracle arithmetic) -- test infrastructure only."""

    def __init__(self, plan: ShardPlan, B: int):
        self.plan = plan
        self.nl = plan.n_local
        self.states = [None] * B

    def half_buffer(self):
        return torch.empty(1 << (self.nl - 1), dtype=torch.complex128)

    def comm_device(self):
        return torch.device("cpu")

    def before_send(self):
        pass

    def after_recv(self):
        pass

    def run_range(self, sel, p0, p1, zero_vector=False):
        prog = self.plan.program
        for b in range(sel.shape[0]):
            if p0 == 0:
                self.states[b] = O.zero_state(self.nl)
                if zero_vector:
                    self.states[b][0] = 0
            psi = self.states[b]
            for p in prog.passes[p0:p1]:
                for i in p.ops:
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
            self.states[b] = psi

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


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = small_circuit()
    plan = plan_sharded(c, 1)
    specs = P.presample_probabilistic(c, 50, 1, np.random.default_rng(4))[:2]
    shard = NumpyShard(plan, len(specs))
    DistributedShards(plan, shard).run(sharded_selection(plan, specs))
    gathered = [None] * world if rank == 0 else None
    dist.gather_object([s.copy() for s in shard.states], gathered, dst=0)
    if rank == 0:
        q.put([[g[b] for g in gathered] for b in range(len(specs))])
    dist.barrier()
    dist.destroy_process_group()


def test_world2_gloo_sharded_state_matches_oracle():
    c = small_circuit()
    plan = plan_sharded(c, 1)
    assert plan.n_swaps >= 1
    specs = P.presample_probabilistic(c, 50, 1, np.random.default_rng(4))[:2]
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    qq = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, qq)) for r in range(2)]
    for p in procs:
        p.start()
    per_traj = qq.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for b, spec in enumerate(specs):
        ref, _ = O.prepare(c, spec.selections)
        got = assemble(plan, per_traj[b])
        assert np.linalg.norm(got - ref) <= 1e-12


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
