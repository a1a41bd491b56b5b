"""Pin the CPU oracle (oracle/engine.py) to golden vectors produced by the reference itself."""

import numpy as np
import pytest

from conftest import build_case
from oracle import engine as O


def test_mix_seed_goldens(golden):
    # ref tests/test_execute.py:11-16 plus extra pairs from make_golden.py
    for m, s, v in golden["mix_seed"]:
        assert O.mix_seed(m, s) == v
    assert O.mix_seed(0, 0) == 16294208416658607535


def test_pcg64_restatement(golden):
    for rec in golden["pcg64"]:
        u = O.pcg64_uniforms(int(rec["state"]), int(rec["inc"]), 8)
        assert np.array_equal(u, np.array(rec["uniforms"]))


@pytest.mark.parametrize("name", ["rychain_mixture", "rychain_damped", "teleport_damped", "ghz4_depol",
                                  "distill5_custom", "config1", "config2", "brick8", "steane1"])
def test_oracle_prepare_and_sample(golden, golden_arrays, name):
    case = golden["cases"][name]
    c = build_case(case)
    for prep in case["prepared"]:
        sel = tuple(tuple(p) for p in prep["selections"])
        if "annihilated" in prep:
            with pytest.raises(O.Annihilated):
                O.prepare(c, sel)
            continue
        psi, w = O.prepare(c, sel)
        ref = golden_arrays[prep["amps"]]
        assert np.linalg.norm(psi - ref) <= 1e-13 * max(1.0, np.linalg.norm(ref))
        assert w == pytest.approx(prep["weight"], rel=1e-13, abs=0)
        m, (ms, st) = prep["sample_m"], prep["sample_seed"]
        rng = np.random.Generator(np.random.PCG64(O.mix_seed(ms, st)))
        assert O.sample(ref, m, rng, c.n_qubits) == prep["counts"]


@pytest.mark.parametrize("name", ["rychain_mixture", "teleport_damped", "config1"])
def test_oracle_dataset_records(golden, name):
    import paper_2504_16297_b200 as P
    case = golden["cases"][name]
    c = build_case(case)
    specs = [P.TrajectorySpec(tuple(tuple(p) for p in t["selections"]), t["shots"], t["joint_prob"], t["tags"])
             for t in case["dataset"]["manifest_core"]["trajectories"]]
    rows = O.run_all(c, specs, case["dataset"]["master_seed"], workers=2)
    recs = []
    for t, row in enumerate(rows):
        recs += [[t, b, row["counts"][b]] for b in sorted(row["counts"])]
    assert recs == case["dataset"]["records"]


def test_coset_oracle_equals_full_state_oracle():
    """oracle.apply_on_cosets (the 28-q pass-parity checker) equals apply_local on the full
    state, restricted to the sampled cosets, for 1q/2q ops inside a scattered qubit set."""
    rng = np.random.default_rng(0)
    n = 10
    psi = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    qubits = [0, 1, 4, 7, 9]
    items = []
    for _ in range(12):
        k = int(rng.integers(1, 3))
        t = [int(x) for x in rng.choice(qubits, size=k, replace=False)]
        m = rng.normal(size=(1 << k, 1 << k)) + 1j * rng.normal(size=(1 << k, 1 << k))
        items.append((m, t))
    full = psi.copy()
    for m, t in items:
        full = O.apply_local(full, m, t, n)
    rest = [q for q in range(n) if q not in qubits]
    pats = np.array([0, 3, 17, 31])
    idx = O.scatter_bits(pats, rest)[:, None] | O.scatter_bits(np.arange(1 << len(qubits)), qubits)[None, :]
    got = O.apply_on_cosets(psi[idx], items, qubits)
    assert np.allclose(got, full[idx], rtol=1e-13, atol=1e-13)


def test_oracle_conventional_trajectories_match_reference_goldens():
    """oracle.run_conventional (trajectory.py:40-70) against the reference's run_trajectory goldens."""
    import json
    from conftest import GOLDEN, build_case
    from paper_2504_16297_b200.execute import stream_rng
    g = json.loads((GOLDEN / "golden_conv.json").read_text())
    with np.load(GOLDEN / "golden_conv.npz") as z:
        arrays = {k: z[k] for k in z.files}
    for name, case in g["cases"].items():
        c = build_case(case)
        for run in case["run_trajectory"]:
            rng = stream_rng(*run["seed"])
            out = O.run_conventional(c, rng)
            assert [list(p) for p in out["selections"]] == run["selections"], name
            assert out["weight"] == pytest.approx(run["weight"], rel=1e-13)
            ref = arrays[run["amps"]]
            assert np.linalg.norm(out["state"] - ref) <= 1e-12 * np.linalg.norm(ref)
            assert float(rng.random()) == run["next_uniform"]
