"""Host-side API surface vs the reference's behaviour (golden vectors + ported unit tests).

Circuit/noise registration, hashes, moments, sites and every PTS strategy must
be bit-identical to the reference (north_star: Kraus assignments bit-exact).
"""

import math

import numpy as np
import pytest

import paper_2504_16297_b200 as P
from paper_2504_16297_b200.errors import CircuitSyntaxError, ValidationError
from conftest import build_case

CASES = ["rychain_mixture", "rychain_damped", "teleport_damped", "ghz4_depol", "distill5_custom",
         "config1", "config2", "brick8", "steane1"]


def spec_json(s):
    return {"selections": [list(p) for p in s.selections], "shots": s.shots,
            "joint_prob": s.joint_prob, "tags": s.tags}


@pytest.mark.parametrize("name", CASES)
def test_structure_and_hashes(golden, name):
    case = golden["cases"][name]
    c = build_case(case)
    assert c.n_qubits == case["n_qubits"]
    assert len(c.ops) == case["n_ops"] and len(c.sites) == case["n_sites"]
    assert list(c.moments) == case["moments"]
    assert [[s.site_id, s.position, s.moment, list(s.targets), s.channel_id] for s in c.sites] == case["sites"]
    assert P.circuit_hash(c) == case["circuit_sha256"]
    from paper_2504_16297_b200.circuit import sites_hash
    assert sites_hash(c) == case["sites_sha256"]
    table = P.site_outcome_probs(c)
    assert [[float(x) for x in e.probs] for e in table] == case["site_probs"]   # bit-exact


@pytest.mark.parametrize("name", CASES)
def test_pts_strategies_bit_exact(golden, name):
    case = golden["cases"][name]
    c = build_case(case)
    pts = case["pts"]
    raw = []
    specs = P.presample_probabilistic(c, 200, 1000, np.random.default_rng(11), raw_sink=raw)
    assert [spec_json(s) for s in specs] == pts["probabilistic"]
    assert [[list(p) for p in r] for r in raw[:50]] == pts["probabilistic_raw"]
    if "filtered" in pts:
        flt = P.SiteFilter(qubits=frozenset({0, 1}))
        got = P.presample_probabilistic(c, 100, 10, np.random.default_rng(5), site_filter=flt)
        assert [spec_json(s) for s in got] == pts["filtered"]
    if "band" in pts:
        got = P.presample_band(c, 1e-4, 0.5, 300, 7, np.random.default_rng(2))
        assert [spec_json(s) for s in got] == pts["band"]
        assert [spec_json(s) for s in P.reallocate_proportional(specs, 12345)] == pts["proportional"]
        got = P.enumerate_cutoff(c, case["cutoff_value"], 50)
        assert [spec_json(s) for s in got] == pts["cutoff"]


def test_vectorised_draws_span_chunks():
    # more samples than one vectorised chunk: stream order must still match scalar draws
    from paper_2504_16297_b200 import presample as PS
    c = P.attach_noise(P.parse_circuit("qubits 2\ngate x 0\ngate x 1\ngate cx 0 1\n"),
                       P.parse_noise_model("rule gate=* qubit=* channel=depolarizing(0.3)\n"))
    a = P.presample_probabilistic(c, PS._CHUNK + 37, 1, np.random.default_rng(4))
    rng = np.random.default_rng(4)
    table = P.site_outcome_probs(c)
    seen, expect = set(), []
    for _ in range(PS._CHUNK + 37):
        sample, p = [], 1.0
        for e in table:
            k = P.select_index(rng.random(), e.probs)
            out = k if k == 0 or P.compatible((e.site.site_id, k), sample, c) else 0
            if out:
                sample.append((e.site.site_id, out))
            p *= float(e.probs[out])
        key = tuple(sample)
        if key not in seen:
            seen.add(key)
            expect.append((key, p))
    assert [(s.selections, s.joint_prob) for s in a] == expect


def test_mix_seed_and_stream_rng():
    from paper_2504_16297_b200.execute import mix_seed, stream_rng
    assert mix_seed(0, 0) == 16294208416658607535
    assert mix_seed(0, 1) == 7960286522194355700
    assert mix_seed(12345, 7) == 7959005890829367068
    assert mix_seed(2**63, 2**32) == 4088906904164161410
    assert stream_rng(3, 4).random() == np.random.Generator(np.random.PCG64(mix_seed(3, 4))).random()


# ---- ported behaviour checks (ref tests/test_circuit.py, test_noise.py, test_presample.py)

@pytest.mark.parametrize("text,message", [
    ("gate h 0\n", "must come before"),
    ("qubits 2\ngate h 5\n", "out of range"),
    ("qubits 2\ngate foo 0\n", "unknown gate"),
    ("qubits 2\ngate cx 0 0\n", "duplicate"),
    ("qubits 2\ngate rx 0 @ abc\n", "bad angle"),
    ("qubits 1\numat 0 : 1 0 0\n", "needs 4 entries"),
    ("qubits 1\numat 0 : 1 1 1 1\n", "not unitary"),
    ("qubits 2\nqubits 3\n", "duplicate 'qubits'"),
    ("qubits 1\nfrobnicate\n", "unknown statement"),
    ("", "missing 'qubits"),
])
def test_parse_errors(text, message):
    with pytest.raises(CircuitSyntaxError, match=message):
        P.parse_circuit(text)


def test_parse_error_line_numbers():
    with pytest.raises(CircuitSyntaxError) as exc:
        P.parse_circuit("qubits 2\n# c\ngate h 9\n")
    assert exc.value.line == 3


@pytest.mark.parametrize("text,message", [
    ("rule gate=h qubit=* channel=nope(0.1)\n", "unknown channel"),
    ("rule gate=h qubit=*\n", "missing key"),
    ("kraus 1 0 0 1\n", "outside a channel"),
    ("channel name=a arity=1\nkraus 1 0\nend\n", "needs 4 entries"),
    ("channel name=a arity=1\nkraus 1 0 0 1\n", "unterminated"),
    ("rule gate=h qubit=* channel=bit_flip(2.0)\n", "must be in"),
])
def test_noise_model_errors(text, message):
    with pytest.raises(CircuitSyntaxError, match=message):
        P.parse_noise_model(text)


def test_noise_model_rejects_non_cptp():
    with pytest.raises(ValidationError, match="trace preserving"):
        P.parse_noise_model("channel name=bad arity=1\nkraus 1 0 0 1\nkraus 1 0 0 1\nend\n"
                            "rule gate=* qubit=* channel=bad\n")


def test_builtin_channels():
    d0 = P.builtin_channel("depolarizing", 0.0)
    assert len(d0.kraus_ops) == 1
    mix = P.builtin_channel("depolarizing", 0.3).unitary_mixture()
    assert np.array_equal(mix.unitaries[0], np.eye(2))          # exact identity: device skips it
    assert P.builtin_channel("amplitude_damping", 0.2).unitary_mixture() is None
    with pytest.raises(ValidationError):
        P.builtin_channel("bit_flip", 1.5)
    assert P.builtin_channel("bit_flip", 0.25).name == "bit_flip(0.25)"


def test_attach_chunking_and_first_match():
    c = P.parse_circuit("qubits 3\ngate h 0\ngate cx 0 1\ngate x 2\n")
    m = P.parse_noise_model("rule gate=cx qubit=* channel=bit_flip(0.1)\nrule gate=* qubit=* channel=phase_flip(0.2)\n")
    nc = P.attach_noise(c, m)
    assert [(s.position, s.targets, s.channel_id) for s in nc.sites] == [
        (0, (0,), "phase_flip(0.2)"), (1, (0,), "bit_flip(0.1)"), (1, (1,), "bit_flip(0.1)"), (2, (2,), "phase_flip(0.2)")]


def test_presample_validation_and_joint_prob():
    c = P.attach_noise(P.parse_circuit("qubits 3\ngate x 0\ngate x 1\ngate x 2\n"),
                       P.parse_noise_model("rule gate=x qubit=* channel=bit_flip(0.1)\n"))
    assert P.joint_probability([], c) == pytest.approx(0.729)
    assert P.joint_probability([(1, 1)], c) == pytest.approx(0.081)
    with pytest.raises(ValidationError, match="duplicate site"):
        P.canonical_selections([(1, 1), (1, 2)])
    with pytest.raises(ValidationError, match="defaults"):
        P.canonical_selections([(1, 0)])
    with pytest.raises(ValidationError, match="nsamples"):
        P.presample_probabilistic(c, 0, 1, np.random.default_rng(0))
    specs = P.enumerate_cutoff(c, 0.05, 10)
    assert [(s.selections, round(s.joint_prob, 12)) for s in specs] == [
        ((), 0.729), (((0, 1),), 0.081), (((1, 1),), 0.081), (((2, 1),), 0.081)]
    with pytest.raises(ValidationError, match="bound"):
        P.enumerate_cutoff(c, 0.0, 10, max_sets=4)


def test_reallocate_proportional_examples():
    specs = [P.TrajectorySpec((), 1, 0.5), P.TrajectorySpec(((0, 1),), 1, 0.25), P.TrajectorySpec(((1, 1),), 1, 0.25)]
    assert [s.shots for s in P.reallocate_proportional(specs, 10)] == [5, 3, 2]
    with pytest.raises(ValidationError, match="no joint"):
        P.reallocate_proportional([P.TrajectorySpec((), 1, None)], 3)
