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
