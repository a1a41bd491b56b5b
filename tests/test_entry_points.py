"""Secondary entry points of the boundary and the CLI, against the reference's own outputs.

``execute_trajectory`` / ``execute_naive`` (ref ``execute.py:101-127``),
``throughput_report`` / ``write_throughput_csv`` (``:320-349``; the deterministic
columns -- m, mode, unique fraction -- since rates are timings),
``kraus_outcome_probability`` on non-trivial states (``statevector.py:129-133``),
and the CLI's ``run`` / ``bench`` files (``cli.py:146-219``).  Golden vectors:
``tests/golden/make_golden_conv.py`` (runs the reference).  Validation, parse
and I/O exit codes need no GPU; everything that executes does (``-m gpu``).
"""

import json

import numpy as np
import pytest

import paper_2504_16297_b200 as P
from paper_2504_16297_b200 import cli
from paper_2504_16297_b200.execute import (execute_naive, execute_trajectory, stream_rng, throughput_report,
                                           write_throughput_csv)
from conftest import GOLDEN, build_case

CASES = ["teleport_damped", "ghz4_depol", "rychain_damped", "brick8_mixed", "ghz10_damped", "config1",
         "brick11_mixed"]


@pytest.fixture(scope="module")
def gconv():
    return json.loads((GOLDEN / "golden_conv.json").read_text())


@pytest.fixture(scope="module")
def gconv_arrays():
    with np.load(GOLDEN / "golden_conv.npz") as z:
        return {k: z[k] for k in z.files}


# ------------------------------------------------------------------ device entry points

@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_execute_trajectory_and_naive_match_reference(gconv, name):
    case = gconv["cases"][name]
    c = build_case(case)
    for i, d in enumerate(case["execute_trajectory"]):
        spec = P.TrajectorySpec(tuple(tuple(p) for p in d["selections"]), d.get("shots", 300))
        if "annihilated" in d:
            with pytest.raises(P.AnnihilatedStateError):
                execute_trajectory(c, spec, stream_rng(13, i))
            continue
        rng = stream_rng(13, i)
        res = execute_trajectory(c, spec, rng)
        assert res.batch.counts == d["counts"]
        assert res.batch.total == spec.shots
        assert res.realized_weight == pytest.approx(d["weight"], rel=1e-12, abs=0)
        assert res.prep_time >= 0 and res.sample_time >= 0
        # the generator advanced by exactly spec.shots draws (statevector.py:161)
        ref_rng = stream_rng(13, i)
        ref_rng.random(spec.shots)
        assert rng.random() == ref_rng.random()
        nb, dt = execute_naive(c, spec, 25, stream_rng(17, i))
        assert nb.counts == d["naive_counts"] and nb.total == d["naive_total"] == 25
        assert dt > 0


@pytest.mark.gpu
def test_throughput_report_and_csv(gconv, tmp_path):
    c = P.attach_noise(P.parse_circuit(gconv_demo("rychain4.circ", gconv)), P.parse_noise_model(
        gconv_demo("rychain_mixture.noise", gconv)))
    spec = P.TrajectorySpec((), 0, None, {"strategy": "bench"})
    rows = throughput_report(c, spec, [1, 10, 100, 1000], master_seed=5, naive_prep_cap=8)
    assert [[r.m, r.mode, r.unique_fraction] for r in rows] == gconv["throughput_rychain"]
    assert all(r.shots_per_second > 0 for r in rows)
    path = write_throughput_csv(rows, tmp_path / "t.csv")
    lines = path.read_text().splitlines()
    assert lines[0] == "m,mode,shots_per_second,unique_fraction"
    for line, r in zip(lines[1:], rows):
        m, mode, sps, uf = line.split(",")
        assert (int(m), mode, float(sps), float(uf)) == (r.m, r.mode, r.shots_per_second, r.unique_fraction)
    with pytest.raises(P.ValidationError):
        throughput_report(c, spec, [0])


def gconv_demo(name, gconv):
    """Demo texts travel inside the golden file (the reference tree is not on the GPU box)."""
    case = gconv["cli"]["run_probabilistic"]
    return case["circuit"] if name.endswith(".circ") else case["noise"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_kraus_outcome_probability_nonzero(gconv, gconv_arrays, name):
    """||K psi||^2 of every Kraus operator of the first sites on the noiseless prepared state."""
    case = gconv["cases"][name]
    c = build_case(case)
    kp = case["kraus_probs"]
    st = P.ComplexState(c.n_qubits, gconv_arrays[kp["amps"]])
    nonzero = 0
    for d in kp["sites"]:
        ch = c.channels[d["channel"]]
        for K, want in zip(ch.kraus_ops, d["probs"]):
            got = P.kraus_outcome_probability(st, K, tuple(d["targets"]))
            assert got == pytest.approx(want, rel=1e-12, abs=1e-15)
            nonzero += want > 1e-6
    assert nonzero >= len(kp["sites"])
    # the state is not mutated (statevector.py:121)
    assert np.array_equal(st.amplitudes, gconv_arrays[kp["amps"]])


# ------------------------------------------------------------------ CLI

def _write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


@pytest.mark.gpu
@pytest.mark.parametrize("cname", ["run_probabilistic", "run_proportional", "run_cutoff_damped",
                                   "run_probabilistic_damped", "run_band_filtered"])
def test_cli_run_matches_reference_files(gconv, cname, tmp_path):
    d = gconv["cli"][cname]
    circ = _write(tmp_path, "c.circ", d["circuit"])
    noise = _write(tmp_path, "n.noise", d["noise"])
    out = tmp_path / "ds"
    code = cli.main(["run", "--circuit", circ, "--noise", noise, "--out", str(out)] + d["argv"])
    assert code == d["code"]
    if code != 0:
        return
    assert (out / "records.jsonl").read_text() == d["records"]
    man = json.loads((out / "manifest.json").read_text())
    got = P.manifest_core(man)
    want = d["manifest_core"]
    for row_g, row_r in zip(got["trajectories"], want["trajectories"]):
        wg, wr = row_g.pop("realized_weight"), row_r.pop("realized_weight")
        assert wg == pytest.approx(wr, rel=1e-12, abs=0)
    assert got == want


@pytest.mark.gpu
def test_cli_bench_matches_reference_files(gconv, tmp_path):
    d = gconv["cli"]["bench"]
    circ = _write(tmp_path, "c.circ", d["circuit"])
    noise = _write(tmp_path, "n.noise", d["noise"])
    out = tmp_path / "b"
    code = cli.main(["bench", "--circuit", circ, "--noise", noise, "--seed", "11", "--out", str(out),
                     "--batch-sizes", "1,10,100,1000", "--naive-prep-cap", "4"])
    assert code == d["code"] == 0
    assert (out / "uniqueness.csv").read_text() == d["uniqueness"]
    thr = [line.split(",") for line in (out / "throughput.csv").read_text().splitlines()]
    assert thr[0] == d["throughput_header"]
    assert [[r[0], r[1], r[3]] for r in thr[1:]] == d["throughput_cols"]


@pytest.mark.gpu
def test_cli_conventional_writes_reference_dataset(gconv, tmp_path):
    case = gconv["cases"]["ghz10_damped"]
    d = case["sample_conventional"]["12x200_s8"]
    circ = _write(tmp_path, "c.circ", case["circuit"])
    noise = _write(tmp_path, "n.noise", case["noise"])
    out = tmp_path / "conv"
    assert cli.main(["conventional", "--circuit", circ, "--noise", noise, "--seed", "8", "--ntraj", "12",
                     "--nshots", "200", "--out", str(out)]) == 0
    ds = P.Dataset.read(out)
    ds.validate()
    assert [[r.trajectory_id, r.bitstring, r.count] for r in ds.records] == d["records"]


def test_cli_validate_and_exit_codes(gconv, tmp_path, capsys):
    """No GPU needed: validate output, parse error (2), invalid channel (3), missing file (5),
    the unavailable density oracle (3)."""
    d = gconv["cli"]["run_probabilistic"]
    circ = _write(tmp_path, "c.circ", d["circuit"])
    noise = _write(tmp_path, "n.noise", d["noise"])
    assert cli.main(["validate", circ, noise]) == 0
    out = capsys.readouterr().out
    assert "unitary mixture" in out and "noise sites: 4" in out
    bad = _write(tmp_path, "bad.noise", "channel name=bad arity=1\nkraus 0.5+0i 0+0i 0+0i 0.5+0i\nend\n"
                                        "rule gate=* qubit=* channel=bad\n")
    assert cli.main(["validate", circ, bad]) == 3
    assert "INVALID" in capsys.readouterr().out
    broken = _write(tmp_path, "broken.circ", "qubits 2\ngate x 5\n")
    assert cli.main(["validate", broken, noise]) == 2
    assert "line 2" in capsys.readouterr().err
    assert cli.main(["validate", str(tmp_path / "missing.circ"), noise]) == 5
    assert cli.main(["oracle", "--circuit", circ, "--dataset", str(tmp_path)]) == 3
    assert cli.main(["run", "--circuit", circ, "--noise", noise, "--strategy", "cutoff", "--seed", "1",
                     "--oracle", "--out", str(tmp_path / "x")]) == 3
