"""World-size-2 gloo run of the trajectory-parallel host logic (no GPU needed).

Each rank runs its block of trajectories with a CPU stand-in for the device
engine (the oracle -- test infrastructure), rank 0 merges by trajectory id; the
result must equal the single-process run exactly, as the reference promises
for any worker count (execute.py:1-5).
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_2504_16297_b200 as P
from paper_2504_16297_b200 import workloads
from paper_2504_16297_b200.distributed import deal, execute_all_distributed, merge, run_distributed
from paper_2504_16297_b200.execute import BatchOutput, dataset_from_output, mix_seed


def oracle_runner(c, specs, master_seed, dtype, rng, ids):
    from oracle import engine as O
    rows = [O.run_trajectory(c, s, master_seed, t) for s, t in zip(specs, ids)]
    idx, cnt, nu, w, st = [], [], [], [], []
    for r in rows:
        keys = sorted(int(b, 2) for b in r["counts"])
        fmt = f"0{c.n_qubits}b"
        idx += keys
        cnt += [r["counts"][format(k, fmt)] for k in keys]
        nu.append(len(keys))
        w.append(r["weight"])
        st.append(0 if r["status"] == "ok" else 2)
    off = np.zeros(len(rows) + 1, dtype=np.int64)
    np.cumsum(nu, out=off[1:])
    z = np.zeros(len(rows))
    return BatchOutput(np.array(w), np.array(st, np.int32), np.array(idx, np.uint64),
                       np.array(cnt, np.uint32), off, z, z)


def _case():
    c = workloads.build(1, P.parse_circuit, P.parse_noise_model, P.attach_noise)
    specs = P.presample_probabilistic(c, 300, 50, np.random.default_rng(2))[:11]
    return c, specs


def _worker(rank, world, port, q, out_dir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c, specs = _case()
    out = run_distributed(c, specs, master_seed=5, runner=oracle_runner)
    if rank == 0:
        q.put((out.weights.tolist(), out.indices.tolist(), out.counts.tolist(), out.offsets.tolist()))
    ds = execute_all_distributed(c, specs, master_seed=5, runner=oracle_runner)
    if rank == 0:
        rp, _ = ds.write(out_dir)
        q.put((rp.read_bytes(), P.manifest_core(ds.manifest)))
    else:
        assert ds is None
    dist.barrier()
    dist.destroy_process_group()


def test_deal_covers_ids_once():
    for n in (0, 1, 7, 16, 101):
        for w in (1, 2, 3, 8):
            got = sorted(t for r in range(w) for t in deal(n, w, r))
            assert got == list(range(n))
            sizes = [len(deal(n, w, r)) for r in range(w)]
            assert max(sizes) - min(sizes) <= 1


def test_world2_gloo_matches_single_process(tmp_path):
    c, specs = _case()
    single = oracle_runner(c, specs, 5, "c128", "pcg64", list(range(len(specs))))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, str(tmp_path / "w2"))) for r in range(2)]
    for p in procs:
        p.start()
    w, idx, cnt, off = q.get(timeout=240)
    records_w2, core_w2 = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert w == single.weights.tolist()
    assert idx == single.indices.tolist() and cnt == single.counts.tolist() and off == single.offsets.tolist()
    # the merged dataset's records.jsonl (native writer) and manifest equal a single-process run's,
    # and the records equal the per-record json.dumps text
    ds1 = dataset_from_output(c, specs, single, master_seed=5)
    rp, _ = ds1.write(tmp_path / "w1")
    assert rp.read_bytes() == records_w2
    assert P.manifest_core(ds1.manifest) == core_w2
    P.Dataset(ds1.manifest, list(ds1.records)).write(tmp_path / "json")
    assert (tmp_path / "json" / "records.jsonl").read_bytes() == records_w2
    assert sum(r["emitted"] for r in core_w2["trajectories"]) == core_w2["total_shots"] > 0


def test_merge_rejects_gaps():
    c, specs = _case()
    a = oracle_runner(c, specs[:2], 0, "c128", "pcg64", [0, 1])
    with pytest.raises(ValueError):
        merge([([0, 2], a)])
