"""CUDA engine vs the reference (golden vectors) and the CPU oracle.

Tolerances (north_star): amplitudes ||psi_dev - psi_ref|| / ||psi_ref|| <= 1e-12
(complex128) / 1e-5 (complex64); realized weights relative 1e-12 / 1e-5;
shots in verification mode (device PCG64 replaying the reference's stream)
exactly equal; Philox-mode histograms pass chi-square at p > 0.01.
"""

import json

import numpy as np
import pytest

import paper_2504_16297_b200 as P
from paper_2504_16297_b200 import _native as N
from paper_2504_16297_b200.engine import Engine, pcg64_state_words
from paper_2504_16297_b200.execute import mix_seed
from paper_2504_16297_b200.program import compile_circuit, selection_matrix
from conftest import build_case
from paper_2504_16297_b200 import workloads
from oracle import engine as O

pytestmark = pytest.mark.gpu

CASES = ["rychain_mixture", "rychain_damped", "teleport_damped", "ghz4_depol", "distill5_custom",
         "config1", "config2", "brick8", "steane1"]
TOL = {"c128": 1e-12, "c64": 1e-5}


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("name", CASES)
def test_prepared_amplitudes_and_weights(golden, golden_arrays, name, dtype):
    case = golden["cases"][name]
    c = build_case(case)
    preps = case["prepared"]
    specs = [P.TrajectorySpec(tuple(tuple(p) for p in d["selections"]), 0) for d in preps]
    with Engine(c.n_qubits, dtype, batch_cap=len(specs)) as eng:
        prog = eng.load(c)
        w, st = eng.run(selection_matrix(prog, specs))
        for b, d in enumerate(preps):
            if "annihilated" in d:
                assert st[b] == N.TRAJ_ANNIHILATED
                continue
            assert st[b] == N.TRAJ_OK
            assert w[b] == pytest.approx(d["weight"], rel=TOL[dtype], abs=0)
            psi = eng.get_state(b)
            assert rel(psi.astype(np.complex128), golden_arrays[d["amps"]]) <= TOL[dtype]


@pytest.mark.parametrize("name", CASES)
def test_shots_bit_exact_pcg64(golden, golden_arrays, name):
    """Verification mode: device replays stream_rng(9, i) -> counts identical to the reference."""
    case = golden["cases"][name]
    c = build_case(case)
    preps = [d for d in case["prepared"] if "annihilated" not in d]
    with Engine(c.n_qubits, "c128", batch_cap=len(preps)) as eng:
        for b, d in enumerate(preps):
            eng.set_state(b, golden_arrays[d["amps"]])
        words = np.concatenate([pcg64_state_words(mix_seed(*d["sample_seed"])) for d in preps])
        out = eng.sample(np.array([d["sample_m"] for d in preps]), N.RNG_PCG64, rng_state=words)
        for b, d in enumerate(preps):
            assert out.counts_dict(b, c.n_qubits) == d["counts"]


@pytest.mark.parametrize("name", ["rychain_mixture", "rychain_damped", "teleport_damped", "config1", "steane1"])
def test_execute_all_records_identical(golden, name, tmp_path):
    """The drop-in boundary: execute_all's records and manifest equal the reference's."""
    case = golden["cases"][name]
    c = build_case(case)
    core = case["dataset"]["manifest_core"]
    specs = [P.TrajectorySpec(tuple(tuple(p) for p in t["selections"]), t["shots"], t["joint_prob"], t["tags"])
             for t in core["trajectories"]]
    ds = P.execute_all(c, specs, parallelism=3, master_seed=case["dataset"]["master_seed"])
    ds.validate()
    assert [[r.trajectory_id, r.bitstring, r.count] for r in ds.records] == case["dataset"]["records"]
    # records.jsonl through the native writer is the reference's json.dumps text
    assert ds.packed is not None
    ds.write(tmp_path)
    want = "".join(json.dumps({"t": t, "b": b, "c": k}, separators=(",", ":")) + "\n"
                   for t, b, k in case["dataset"]["records"])
    assert (tmp_path / "records.jsonl").read_text() == want
    got = P.manifest_core(ds.manifest)
    for row_g, row_r in zip(got["trajectories"], core["trajectories"]):
        wg, wr = row_g.pop("realized_weight"), row_r.pop("realized_weight")
        assert wg == pytest.approx(wr, rel=1e-12, abs=0)
    assert got == core


def test_philox_histograms_chi_square(golden, golden_arrays):
    from scipy import stats
    case = golden["cases"]["config1"]
    c = build_case(case)
    preps = [d for d in case["prepared"] if "annihilated" not in d][:4]
    m = 200_000
    with Engine(c.n_qubits, "c64", batch_cap=len(preps)) as eng:
        for b, d in enumerate(preps):
            eng.set_state(b, golden_arrays[d["amps"]])
        seeds = np.array([mix_seed(5, b) for b in range(len(preps))], dtype=np.uint64)
        out = eng.sample(np.full(len(preps), m), N.RNG_PHILOX, rng_state=seeds)
        for b, d in enumerate(preps):
            probs = np.abs(golden_arrays[d["amps"]]) ** 2
            lo, hi = out.offsets[b], out.offsets[b + 1]
            obs = np.zeros(probs.size)
            obs[out.indices[lo:hi].astype(np.int64)] = out.counts[lo:hi]
            assert obs.sum() == m
            assert np.all(probs[obs > 0] > 0)          # never a zero-probability outcome
            keep = probs * m >= 5
            exp = probs[keep] * m
            o = obs[keep]
            # fold the rare tail into one bin
            o = np.append(o, m - o.sum())
            exp = np.append(exp, m - exp.sum())
            nz = exp > 0
            p = stats.chisquare(o[nz], exp[nz] * o[nz].sum() / exp[nz].sum()).pvalue
            assert p > 0.01


def test_bench20_state_and_shots(golden):
    g = golden["bench20"]
    c = P.parse_circuit(g["circuit"])
    with Engine(20, "c128", batch_cap=1) as eng:
        eng.load(c)
        w, st = eng.run(np.zeros((1, 0), dtype=np.uint8))
        psi = eng.get_state(0)
        probs = np.abs(psi) ** 2
        assert np.allclose(probs.reshape(-1, 1024).sum(axis=1), g["prob_sum_by_1024"], rtol=1e-11, atol=1e-15)
        head = np.array([complex(a, b) for a, b in g["amps_head"]])
        assert np.allclose(psi[:64], head, rtol=1e-11, atol=1e-14)
        out = eng.sample([1000], N.RNG_PCG64, rng_state=pcg64_state_words(mix_seed(0, 0)))
        assert out.counts_dict(0, 20) == g["counts_m1000_seed00"]


def test_uneven_shots_zero_shots_and_annihilation(tmp_path):
    c = P.attach_noise(P.parse_circuit("qubits 3\ngate h 0\ngate cx 0 1\ngate x 2\n"),
                       P.parse_noise_model("rule gate=x qubit=* channel=amplitude_damping(0.5)\n"
                                           "rule gate=* qubit=* channel=depolarizing(0.2)\n"))
    specs = [P.TrajectorySpec((), 0), P.TrajectorySpec(((3, 1),), 7), P.TrajectorySpec(((0, 2),), 1),
             P.TrajectorySpec((), 50_000)]
    ds = P.execute_all(c, specs, master_seed=4)
    ds.validate()
    rows = ds.manifest["trajectories"]
    assert [r["emitted"] for r in rows] == [0, 7, 1, 50_000]
    # K1 of damping on |1> is allowed; on |0> (qubit 2 flipped by x -> |1>) check the annihilating case
    c2 = P.attach_noise(P.parse_circuit("qubits 1\ngate i 0\n"),
                        P.parse_noise_model("rule gate=i qubit=* channel=amplitude_damping(0.5)\n"))
    ds2 = P.execute_all(c2, [P.TrajectorySpec((), 50), P.TrajectorySpec(((0, 1),), 50)], master_seed=0)
    ds2.validate()
    r = ds2.manifest["trajectories"]
    assert ds2.manifest["partial"]
    assert r[0]["status"] == "ok" and r[0]["emitted"] == 50
    assert r[1]["status"] == "annihilated" and r[1]["emitted"] == 0
    for d, sub in ((ds, "a"), (ds2, "b")):    # native writer == per-record json path
        assert d.packed is not None
        d.write(tmp_path / sub / "native")
        P.Dataset(d.manifest, d.records).write(tmp_path / sub / "json")
        assert ((tmp_path / sub / "native" / "records.jsonl").read_bytes()
                == (tmp_path / sub / "json" / "records.jsonl").read_bytes())
    with pytest.raises(P.AnnihilatedStateError):
        P.prepare_state(c2, P.TrajectorySpec(((0, 1),), 1))


def test_general_channel_weight_known_answer():
    # ref tests/test_execute.py:59-68: damping(0.36) after h -> weight 0.82
    c = P.attach_noise(P.parse_circuit("qubits 1\ngate h 0\n"),
                       P.parse_noise_model("rule gate=h qubit=* channel=amplitude_damping(0.36)\n"))
    st, w = P.prepare_state(c, P.TrajectorySpec((), 0))
    assert w == pytest.approx(0.82, rel=1e-12)
    assert st.probabilities()[1] == pytest.approx(0.5 * 0.64 / 0.82, rel=1e-12)


def test_inner_api_matches_reference_semantics():
    s = P.apply_gate(P.init_zero(2), P.gate_op("x", [0]))
    s = P.apply_gate(s, P.gate_op("cx", [0, 1]))
    assert np.allclose(s.probabilities(), [0, 0, 0, 1])
    damp = P.builtin_channel("amplitude_damping", 0.3)
    one = P.apply_gate(P.init_zero(1), P.gate_op("x", [0]))
    out, r = P.apply_kraus_normalized(one, damp.kraus_ops[1], [0])
    assert r == pytest.approx(0.3, rel=1e-12) and np.allclose(out.amplitudes, [1, 0])
    assert P.kraus_outcome_probability(P.init_zero(1), damp.kraus_ops[1], [0]) == pytest.approx(0.0)
    with pytest.raises(P.AnnihilatedStateError):
        P.apply_kraus_normalized(P.init_zero(1), damp.kraus_ops[1], [0])
    # stream concatenation (ref tests/test_statevector.py:145-151)
    st = P.apply_gate(P.init_zero(3), P.gate_op("h", [1]))
    before = st.amplitudes.copy()
    split, whole = np.random.default_rng(9), np.random.default_rng(9)
    merged = P.sample_shots(st, 400, split).merged(P.sample_shots(st, 600, split))
    assert merged.counts == P.sample_shots(st, 1000, whole).counts
    assert np.array_equal(st.amplitudes, before)
    # identical to the oracle's numpy sampler for a random state
    rng = np.random.default_rng(42)
    amps = rng.normal(size=256) + 1j * rng.normal(size=256)
    amps /= np.linalg.norm(amps)
    dev = P.sample_shots(P.ComplexState(8, amps), 20_000, np.random.default_rng(3)).counts
    assert dev == O.sample(amps, 20_000, np.random.default_rng(3), 8)
    with pytest.raises(P.ValidationError, match=">= 1"):
        P.sample_shots(P.init_zero(1), 0, np.random.default_rng(0))


@pytest.mark.parametrize("n", [1, 2, 3, 5])
def test_tiny_states(n):
    ops = "".join(f"gate h {q}\n" for q in range(n))
    c = P.parse_circuit(f"qubits {n}\n{ops}")
    for dtype in ("c64", "c128"):
        with Engine(n, dtype, batch_cap=2) as eng:
            eng.load(c)
            eng.run(np.zeros((2, 0), dtype=np.uint8))
            psi = eng.get_state(1)
            assert np.allclose(psi, np.full(1 << n, 2 ** (-n / 2)), atol=1e-6)
            out = eng.sample([1000, 3], N.RNG_PHILOX, rng_state=np.array([1, 2], dtype=np.uint64))
            assert out.counts[: out.offsets[1]].sum() == 1000 and out.counts[out.offsets[1]:].sum() == 3
    empty = P.parse_circuit(f"qubits {n}\n")
    st, w = P.prepare_state(empty, P.TrajectorySpec((), 0))
    assert st.amplitudes[0] == 1 and w == 1.0


def test_tile_sizes_agree_at_22_qubits():
    """Size-independent property: different fusion plans give the same state (c128)."""
    c = P.parse_circuit(workloads.random_brickwork(22, layers=4, seed=9)[0])
    states = []
    for tb in (8, 10, 12):
        prog = compile_circuit(c, "c128", tile_bits=tb)
        with Engine(22, "c128", batch_cap=1) as eng:
            eng.load_program(prog)
            eng.run(np.zeros((1, 0), dtype=np.uint8))
            states.append(eng.get_state(0))
    assert rel(states[0], states[1]) <= 1e-12 and rel(states[2], states[1]) <= 1e-12
    assert abs(np.linalg.norm(states[1]) - 1) <= 1e-12


def test_config3_20q_against_oracle():
    c = workloads.build(3, P.parse_circuit, P.parse_noise_model, P.attach_noise)
    specs = P.presample_probabilistic(c, 30, 100, np.random.default_rng(1))[:2]
    for dtype in ("c128", "c64"):
        with Engine(20, dtype, batch_cap=2) as eng:
            prog = eng.load(c)
            w, st = eng.run(selection_matrix(prog, specs))
            assert len(specs) == 2
            for b, s in enumerate(specs):
                ref, rw = O.prepare(c, s.selections)
                assert st[b] == 0 and w[b] == pytest.approx(rw, rel=TOL[dtype], abs=0)
                assert rel(eng.get_state(b).astype(np.complex128), ref) <= TOL[dtype]


def test_config4_28q_properties():
    """Full-size config 4 (28 q, c64): norm, determinism, shot totals, no zero-probability outcomes."""
    c = workloads.build(4, P.parse_circuit, P.parse_noise_model, P.attach_noise)
    specs = P.presample_probabilistic(c, 20, 10_000, np.random.default_rng(3))[:2]
    with Engine(28, "c64", batch_cap=2) as eng:
        prog = eng.load(c)
        sel = selection_matrix(prog, specs)
        w, st = eng.run(sel)
        assert list(st) == [0, 0] and np.allclose(w, 1.0)
        words = np.concatenate([pcg64_state_words(mix_seed(1, t)) for t in range(2)])
        a = eng.sample([10_000, 10_000], N.RNG_PCG64, rng_state=words)
        eng.run(sel)
        b = eng.sample([10_000, 10_000], N.RNG_PCG64, rng_state=words)
        assert np.array_equal(a.indices, b.indices) and np.array_equal(a.counts, b.counts)
        assert int(a.counts.sum()) == 20_000
        assert a.indices.max() < (1 << 28)
        psi = eng.get_state(0)
        assert abs(float(np.sum(np.abs(psi.astype(np.complex128)) ** 2)) - 1.0) < 1e-4
        assert np.all(np.abs(psi[a.indices[: a.offsets[1]].astype(np.int64)]) > 0)


def test_permuted_layout_sampling_modes():
    """Config 2 (17 q, c128) is planned with a permuted physical layout: PCG64 shots must still
    equal the reference sampler on the logical state, Philox shots must follow |psi|^2."""
    from scipy import stats
    c = workloads.build(2, P.parse_circuit, P.parse_noise_model, P.attach_noise)
    specs = P.enumerate_cutoff(c, 1e-5, 4000)[:3]
    with Engine(17, "c128", batch_cap=3) as eng:
        prog = eng.load(c)
        assert prog.perm != list(range(17))
        sel = selection_matrix(prog, specs)
        eng.run(sel)
        seeds = np.array([mix_seed(7, t) for t in range(3)], dtype=np.uint64)
        ph = eng.sample([s.shots for s in specs], N.RNG_PHILOX, rng_state=seeds)
        words = np.concatenate([pcg64_state_words(mix_seed(7, t)) for t in range(3)])
        ex = eng.sample([s.shots for s in specs], N.RNG_PCG64, rng_state=words)
        for b, s in enumerate(specs):
            ref, _ = O.prepare(c, s.selections)
            assert rel(eng.get_state(b), ref) <= 1e-12
            rng = np.random.Generator(np.random.PCG64(mix_seed(7, b)))
            assert ex.counts_dict(b, 17) == O.sample(ref, s.shots, rng, 17)
            lo, hi = ph.offsets[b], ph.offsets[b + 1]
            idx = ph.indices[lo:hi].astype(np.int64)
            assert np.all(np.diff(idx) > 0) and int(ph.counts[lo:hi].sum()) == s.shots
            probs = np.abs(ref) ** 2
            assert np.all(probs[idx] > 0)
            top = np.argsort(probs)[::-1][:8]
            obs = np.array([ph.counts[lo:hi][idx == t].sum() for t in top], dtype=float)
            exp = probs[top] * s.shots
            obs = np.append(obs, s.shots - obs.sum())
            exp = np.append(exp, s.shots - exp.sum())
            assert stats.chisquare(obs, exp).pvalue > 0.01


@pytest.mark.parametrize("cfg,dtype", [(2, "c128"), (4, "c64")])
def test_shared_trunk_schedule_is_bit_identical(cfg, dtype, monkeypatch):
    """Forking trajectories off the shared noiseless trunk must give exactly the states of
    evolving each one from |0> on its own (PTSBE_TREE=0)."""
    c = workloads.build(cfg, P.parse_circuit, P.parse_noise_model, P.attach_noise)
    specs = P.presample_probabilistic(c, 400, 10, np.random.default_rng(8))[:5]
    prog = compile_circuit(c, dtype)
    assert prog.n_passes >= 2
    out = {}
    for tree in ("1", "0"):
        monkeypatch.setenv("PTSBE_TREE", tree)
        with Engine(c.n_qubits, dtype, batch_cap=len(specs)) as eng:
            eng.load_program(prog)
            w, st = eng.run(selection_matrix(prog, specs))
            out[tree] = (w, st, [eng.get_state(b) for b in range(len(specs))])
    assert np.array_equal(out["1"][0], out["0"][0]) and np.array_equal(out["1"][1], out["0"][1])
    for a, b in zip(out["1"][2], out["0"][2]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("cfg,dtype", [(3, "c64"), (4, "c64"), (4, "c128")])
def test_circuit_specialised_kernels_are_active(cfg, dtype):
    """The generated (NVRTC) pass kernels compile and load for the bench-size programs: the
    generic interpreter kernel is a correctness fallback only, it must not be what runs."""
    c = workloads.build(cfg, P.parse_circuit, P.parse_noise_model, P.attach_noise)
    with Engine(c.n_qubits, dtype, batch_cap=1) as eng:
        eng.load(c)
        assert eng.info()["codegen"] == 1


@pytest.mark.parametrize("fused,dtype", [(True, "c64"), (False, "c64"), (True, "c128"), (False, "c128")])
def test_fused_block_sums_philox_chi_square(fused, dtype, monkeypatch):
    """Config 3 (20 q, c64, generated kernels, unitary mixtures): the last pass writes the
    sampler's block sums in its tile order (no separate state read); Philox shots drawn on that
    CDF must still follow |psi|^2 of the logical state, exactly like the index-order path."""
    from scipy import stats
    if not fused:
        monkeypatch.setenv("PTSBE_NO_FUSED_SUMS", "1")
    c = workloads.build(3, P.parse_circuit, P.parse_noise_model, P.attach_noise)
    specs = P.presample_probabilistic(c, 30, 100, np.random.default_rng(1))[:2]
    m = 400_000
    with Engine(20, dtype, batch_cap=2) as eng:
        prog = eng.load(c)
        assert eng.info()["codegen"] == 1
        eng.run(selection_matrix(prog, specs))
        seeds = np.array([mix_seed(11, t) for t in range(2)], dtype=np.uint64)
        out = eng.sample(np.full(2, m), N.RNG_PHILOX, rng_state=seeds)
        for b in range(2):
            probs = np.abs(eng.get_state(b).astype(np.complex128)) ** 2
            lo, hi = out.offsets[b], out.offsets[b + 1]
            idx = out.indices[lo:hi].astype(np.int64)
            assert np.all(np.diff(idx) > 0)                  # ascending, distinct (ShotBatch order)
            obs = np.zeros(probs.size)
            obs[idx] = out.counts[lo:hi]
            assert obs.sum() == m
            assert np.all(probs[obs > 0] > 0)
            # a 20-q random state is spread over ~10^6 outcomes (Porter-Thomas): test the
            # marginals of the high and the low 10 qubits (1024 bins each, ~400 shots per bin),
            # which a wrong tile-order -> basis-index mapping would scramble
            # alpha = 1e-3 per test, the reference's level for its batched-fidelity chi^2
            # (test_execute.py:168-178): 4 params x 2 trajectories x 2 marginals = 16 tests
            # at 0.01 would fail by chance ~15 % of the time (seen: p = 0.007, c128, seed 11,
            # trajectory 1; other seeds and 4x the shots give p = 0.2-0.98)
            for fold in (lambda v: v.reshape(1024, -1).sum(axis=1), lambda v: v.reshape(-1, 1024).sum(axis=0)):
                o, exp = fold(obs), fold(probs) * m
                p = stats.chisquare(o, exp * o.sum() / exp.sum()).pvalue
                assert p > 1e-3


def test_execute_all_distributed_single_rank_equals_execute_all(tmp_path):
    """World of one (no process group): the trajectory-parallel driver's Dataset is execute_all's."""
    from paper_2504_16297_b200.distributed import execute_all_distributed
    c = workloads.build(1, P.parse_circuit, P.parse_noise_model, P.attach_noise)
    specs = P.presample_probabilistic(c, 200, 300, np.random.default_rng(9))[:20]
    a = P.execute_all(c, specs, master_seed=3)
    b = execute_all_distributed(c, specs, master_seed=3)
    a.write(tmp_path / "a")
    b.write(tmp_path / "b")
    assert (tmp_path / "a" / "records.jsonl").read_bytes() == (tmp_path / "b" / "records.jsonl").read_bytes()
    assert P.manifest_core(a.manifest) == P.manifest_core(b.manifest)
    b.validate()


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_tree_schedule_shared_prefixes_splits_and_duplicates(dtype, monkeypatch):
    """The shared-prefix tree schedule with groups that share several errors, split in the middle
    of the program (owner kept in place after the others read it), renormalising sites and
    duplicated outcome tables (copied at the end) equals independent evolution bit for bit."""
    from paper_2504_16297_b200.program import prefix_order, site_passes
    c = workloads.build(3, P.parse_circuit, P.parse_noise_model, P.attach_noise)
    prog = compile_circuit(c, dtype)
    sp = site_passes(prog)
    by_pass = [[s for s in range(prog.n_sites) if sp[s] == p] for p in range(prog.n_passes)]
    a, b2, b3 = by_pass[0][0], by_pass[1][2], by_pass[prog.n_passes - 1][1]
    sel = [(), ((a, 1),), ((a, 1), (b2, 2)), ((a, 1), (b2, 2), (b3, 1)), ((a, 1), (b2, 3)), ((b2, 2),),
           ((a, 1), (b2, 2)), ()]
    specs = [P.TrajectorySpec(tuple(sorted(x)), 10) for x in sel]
    order = prefix_order(prog, specs)
    assert sorted(order) == list(range(len(specs)))
    out = {}
    for tree in ("1", "0"):
        monkeypatch.setenv("PTSBE_TREE", tree)
        with Engine(c.n_qubits, dtype, batch_cap=len(specs)) as eng:
            eng.load_program(prog)
            w, st = eng.run(selection_matrix(prog, specs))
            words = np.concatenate([pcg64_state_words(mix_seed(3, t)) for t in range(len(specs))])
            shots = eng.sample([200] * len(specs), N.RNG_PCG64, rng_state=words)   # order-independent exact CDF
            out[tree] = (w, st, [eng.get_state(b) for b in range(len(specs))], shots)
    assert np.array_equal(out["1"][0], out["0"][0]) and np.array_equal(out["1"][1], out["0"][1])
    for x, y in zip(out["1"][2], out["0"][2]):
        assert np.array_equal(x, y)
    assert np.array_equal(out["1"][3].indices, out["0"][3].indices)
    assert np.array_equal(out["1"][3].counts, out["0"][3].counts)
    # and against the oracle
    for b, spec in enumerate(specs):
        ref, _ = O.prepare(c, spec.selections)
        assert rel(out["1"][2][b].astype(np.complex128), ref) <= TOL[dtype]


def test_tree_schedule_renormalising_groups(monkeypatch):
    """Groups sharing amplitude-damping outcomes (renormalising, weights inherited at splits)."""
    text = "qubits 6\n" + "".join(f"gate h {q}\ngate ry {q} @ 0.{q + 3}\n" for q in range(6)) + \
        "".join(f"gate cx {q} {q + 1}\n" for q in range(5)) + "".join(f"gate rx {q} @ 1.1\n" for q in range(6))
    c = P.attach_noise(P.parse_circuit(text), P.parse_noise_model("rule gate=* qubit=* channel=amplitude_damping(0.2)\n"))
    prog = compile_circuit(c, "c128", tile_bits=4, low_bits=2)
    assert prog.n_passes >= 3
    S = prog.n_sites
    specs = [P.TrajectorySpec(x, 5) for x in [(), ((0, 1),), ((0, 1), (S - 1, 1)), ((0, 1), (S - 2, 1)),
                                              ((3, 1),), ((0, 1), (S - 1, 1))]]
    out = {}
    for tree in ("1", "0"):
        monkeypatch.setenv("PTSBE_TREE", tree)
        with Engine(c.n_qubits, "c128", batch_cap=len(specs)) as eng:
            eng.load_program(prog)
            w, st = eng.run(selection_matrix(prog, specs))
            out[tree] = (w, st, [eng.get_state(b) for b in range(len(specs))])
    assert np.array_equal(out["1"][0], out["0"][0]) and np.array_equal(out["1"][1], out["0"][1])
    for b, (x, y) in enumerate(zip(out["1"][2], out["0"][2])):
        assert np.array_equal(x, y)
        if out["1"][1][b] == 0:
            ref, rw = O.prepare(c, specs[b].selections)
            assert rel(x, ref) <= 1e-12 and out["1"][0][b] == pytest.approx(rw, rel=1e-12)


def test_tma_issue_forms_and_team_tail_barrier_are_bit_identical(monkeypatch):
    """Steane blocks at 21 q (c128: generated TMA passes, compute teams on the heavy ones): the
    per-lane TMA issue (default), the warp-uniform issue from the __constant__ row table
    (PTSBE_TMA_LANES=0) and the team barrier after every store (PTSBE_TEAM_TAIL_SYNC=1) must
    give exactly the same states and weights."""
    ctext, ntext = workloads.steane_blocks(3)
    c = P.attach_noise(P.parse_circuit(ctext), P.parse_noise_model(ntext))
    specs = P.presample_probabilistic(c, 200, 10, np.random.default_rng(21))[:4]
    prog = compile_circuit(c, "c128")
    out = {}
    for name, env in (("default", {}), ("warp", {"PTSBE_TMA_LANES": "0"}), ("tail", {"PTSBE_TEAM_TAIL_SYNC": "1"})):
        for k in ("PTSBE_TMA_LANES", "PTSBE_TEAM_TAIL_SYNC"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        with Engine(c.n_qubits, "c128", batch_cap=len(specs)) as eng:
            eng.load_program(prog)
            assert eng.info()["codegen"] == 1
            w, st = eng.run(selection_matrix(prog, specs))
            out[name] = (w, st, [eng.get_state(b) for b in range(len(specs))])
    ref = out["default"]
    assert all(abs(np.linalg.norm(s) - 1) <= 1e-12 for s in ref[2])
    for name in ("warp", "tail"):
        assert np.array_equal(out[name][0], ref[0]) and np.array_equal(out[name][1], ref[1])
        for a, b in zip(out[name][2], ref[2]):
            assert np.array_equal(a, b)
