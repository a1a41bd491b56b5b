"""Host/device overlap paths: PTS drawn on a host thread while device
batches run, and the device-resident bench path that never drains the stream.  Both must give
exactly what the plain calls give."""

import numpy as np
import pytest

import paper_2504_16297_b200 as P
from paper_2504_16297_b200 import _native as N
from paper_2504_16297_b200 import workloads
from paper_2504_16297_b200.execute import execute_all, presample_and_execute, stream_rng

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("config,batch", [(1, 7), (2, 16), (1, None)])
def test_presample_and_execute_equals_presample_then_execute_all(config, batch, tmp_path):
    c = workloads.build(config, P.parse_circuit, P.parse_noise_model, P.attach_noise)
    specs_ref = P.presample_probabilistic(c, 3000, 200, stream_rng(4, 2**63))
    ref = execute_all(c, specs_ref, master_seed=4)
    specs, ds = presample_and_execute(c, 3000, 200, stream_rng(4, 2**63), master_seed=4, batch=batch)
    assert specs == specs_ref
    assert [(r.trajectory_id, r.bitstring, r.count) for r in ds.records] == \
        [(r.trajectory_id, r.bitstring, r.count) for r in ref.records]
    a, b = P.manifest_core(ds.manifest), P.manifest_core(ref.manifest)
    assert a == b
    ds.write(tmp_path / "a")
    ref.write(tmp_path / "b")
    assert (tmp_path / "a" / "records.jsonl").read_bytes() == (tmp_path / "b" / "records.jsonl").read_bytes()


def test_device_pointer_path_with_host_mirror_equals_host_path():
    """run_device / sample_device with the host mirror (no read-back, no drain; CSR compacted on
    device) give the host-pointer results bit for bit, over several back-to-back batches."""
    import torch
    from paper_2504_16297_b200.engine import Engine
    from paper_2504_16297_b200.execute import mix_seed
    from paper_2504_16297_b200.program import selection_matrix
    c = workloads.build(3, P.parse_circuit, P.parse_noise_model, P.attach_noise)
    specs = P.presample_probabilistic(c, 400, 3000, np.random.default_rng(1))[:24]
    B = 8
    with Engine(c.n_qubits, "c64", batch_cap=B) as eng:
        prog = eng.load(c)
        sel = selection_matrix(prog, specs)
        shots = np.array([s.shots for s in specs], dtype=np.int64)
        seeds = np.array([mix_seed(9, t) for t in range(len(specs))], dtype=np.uint64)
        want = []
        for lo in range(0, len(specs), B):
            w, st = eng.run(sel[lo:lo + B])
            out = eng.sample(shots[lo:lo + B], N.RNG_PHILOX, rng_state=seeds[lo:lo + B])
            want.append((w, st, out))
        dev = torch.device("cuda", 0)
        d_sel = torch.from_numpy(sel).to(dev)
        d_shots = torch.from_numpy(shots).to(dev)
        d_rng = torch.from_numpy(seeds.view(np.int64)).to(dev)
        d_w = torch.empty(B, dtype=torch.float64, device=dev)
        d_s = torch.empty(B, dtype=torch.int32, device=dev)
        got = []
        for lo in range(0, len(specs), B):
            d_idx = torch.empty(B * 3000, dtype=torch.int64, device=dev)
            d_cnt = torch.empty(B * 3000, dtype=torch.int32, device=dev)
            d_nu = torch.empty(B, dtype=torch.int64, device=dev)
            eng.set_host_mirror(sel[lo:lo + B], shots[lo:lo + B])
            eng.run_device(d_sel.data_ptr() + lo * sel.shape[1], B, d_w.data_ptr(), d_s.data_ptr(), mirror=True)
            eng.sample_device(B, d_shots.data_ptr() + lo * 8, N.RNG_PHILOX, d_rng.data_ptr() + lo * 8,
                              d_idx.data_ptr(), d_cnt.data_ptr(), d_nu.data_ptr(), mirror=True)
            eng.synchronize()
            nu = d_nu.cpu().numpy()
            U = int(nu.sum())
            got.append((d_w.cpu().numpy().copy(), d_s.cpu().numpy().copy(), nu,
                        d_idx[:U].cpu().numpy().view(np.uint64), d_cnt[:U].cpu().numpy().view(np.uint32)))
        for (w, st, out), (gw, gs, nu, idx, cnt) in zip(want, got):
            assert np.array_equal(w, gw) and np.array_equal(st, gs)
            assert np.array_equal(np.diff(out.offsets), nu)
            assert np.array_equal(out.indices, idx) and np.array_equal(out.counts, cnt)
