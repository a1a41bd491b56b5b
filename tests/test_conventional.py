"""Conventional trajectories (Algorithm 1) on the device vs the reference's own outputs.

Golden vectors: ``tests/golden/make_golden_conv.py`` runs the reference's
``run_trajectory`` (``trajectory.py:40-70``) and ``sample_conventional``
(``:73-106``, dense-ensemble path for n <= 8 and per-trajectory streams above)
on circuits with general (amplitude damping) and unitary-mixture channels.

Tolerances (north_star): selections and shot counts identical, weights and
amplitudes relative 1e-12 (complex128) / 1e-5 (complex64).
"""

import json

import numpy as np
import pytest

import paper_2504_16297_b200 as P
from paper_2504_16297_b200 import _native as N
from paper_2504_16297_b200.engine import Engine
from paper_2504_16297_b200.execute import stream_rng
from paper_2504_16297_b200.program import compile_circuit
from paper_2504_16297_b200.trajectory import run_trajectory, sample_conventional
from conftest import GOLDEN, build_case
from oracle import engine as O

pytestmark = pytest.mark.gpu

TOL = {"c128": 1e-12, "c64": 1e-5}
CASES = ["teleport_damped", "ghz4_depol", "rychain_damped", "brick8_mixed", "ghz10_damped", "config1",
         "brick11_mixed"]


@pytest.fixture(scope="module")
def gconv():
    return json.loads((GOLDEN / "golden_conv.json").read_text())


@pytest.fixture(scope="module")
def gconv_arrays():
    with np.load(GOLDEN / "golden_conv.npz") as z:
        return {k: z[k] for k in z.files}


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("name", CASES)
def test_run_trajectory_matches_reference(gconv, gconv_arrays, name, dtype):
    """Same uniforms -> same per-site selections (general sites chosen on device from the
    state), same realized weight and final state; the stream is left where the reference leaves it."""
    case = gconv["cases"][name]
    c = build_case(case)
    for run in case["run_trajectory"]:
        rng = stream_rng(*run["seed"])
        tr = run_trajectory(c, rng, dtype=dtype)
        assert [list(p) for p in tr.selections] == run["selections"]
        assert tr.weight == pytest.approx(run["weight"], rel=TOL[dtype], abs=0)
        assert rel(tr.final_state.amplitudes, gconv_arrays[run["amps"]]) <= TOL[dtype]
        assert float(rng.random()) == run["next_uniform"]


@pytest.mark.parametrize("name", CASES)
def test_sample_conventional_dataset_matches_reference(gconv, name):
    """sample_conventional's records (trajectory, bitstring, count) and manifest equal the
    reference's, for 1 shot and 200 shots per trajectory (both stream orders)."""
    case = gconv["cases"][name]
    c = build_case(case)
    for key, d in case["sample_conventional"].items():
        ds = sample_conventional(c, d["n_traj"], d["shots"], master_seed=d["master_seed"])
        ds.validate()
        assert [[r.trajectory_id, r.bitstring, r.count] for r in ds.records] == d["records"], key
        got = P.manifest_core(ds.manifest)
        want = json.loads(json.dumps(d["manifest_core"]))
        for row_g, row_r in zip(got["trajectories"], want["trajectories"]):
            wg, wr = row_g.pop("realized_weight"), row_r.pop("realized_weight")
            assert wg == pytest.approx(wr, rel=1e-12, abs=0)
        assert json.loads(json.dumps(got)) == want, key


def test_device_branch_probabilities_equal_kraus_norms(gconv):
    """ptsbe_run_conventional's fused multi-branch probabilities (reduced density matrix of the
    site's targets) equal ||K_k psi||^2 of the oracle on the state before the site, at 1e-12."""
    case = gconv["cases"]["ghz10_damped"]
    c = build_case(case)
    prog = compile_circuit(c, "c128", decide_general=True)
    rng = np.random.default_rng(7)
    B = 3
    S = prog.n_sites
    U = rng.random((B, S))
    with Engine(c.n_qubits, "c128", batch_cap=B) as eng:
        eng.load_program(prog)
        sel0 = np.zeros((B, S), dtype=np.uint8)
        out, w, st, probs = eng.run_conventional(sel0, U, with_probs=True)
        assert np.all(st == 0)
        dec = [prog.stream[p.ops[0]] for p in prog.passes if prog.stream[p.ops[0]].general]
        for b in range(B):
            chosen = {sid: int(out[b, sid]) for sid in range(S)}
            psi = O.zero_state(c.n_qubits)
            i_dec = 0
            for mat, targets, general, sid in _stream_with_ids(c, chosen):
                if general:
                    ch = c.channels[c.site(sid).channel_id]
                    want = [float(np.sum(np.abs(O.apply_local(psi, K, targets, c.n_qubits)) ** 2))
                            for K in ch.kraus_ops]
                    assert dec[i_dec].ref == sid
                    got = probs[i_dec, b, :len(want)]
                    assert np.allclose(got, want, rtol=1e-12, atol=1e-15)
                    i_dec += 1
                psi = O.apply_local(psi, mat, targets, c.n_qubits)
                if general:
                    psi = psi / np.linalg.norm(psi)
            assert i_dec == len(dec)


def _stream_with_ids(c, chosen):
    """The reference op loop (execute.py:85-97) with site ids: (matrix, targets, general, site|None)."""
    by_pos = c.sites_by_position()
    for pos, op in enumerate(c.ops):
        yield op.matrix, op.targets, False, None
        for site in by_pos.get(pos, ()):
            ch = c.channels[site.channel_id]
            k = chosen.get(site.site_id, 0)
            mix = ch.unitary_mixture()
            if mix is not None:
                yield mix.unitaries[k], site.targets, False, site.site_id
            else:
                yield ch.kraus_ops[k], site.targets, True, site.site_id


def test_conventional_mode_rejects_unplanned_program():
    """A program whose general sites do not open their passes is refused (no silent PTSBE run)."""
    c = P.attach_noise(P.parse_circuit("qubits 3\ngate h 0\ngate cx 0 1\ngate x 2\n"),
                       P.parse_noise_model("rule gate=* qubit=* channel=amplitude_damping(0.1)\n"))
    prog = compile_circuit(c, "c128")
    with Engine(3, "c128", batch_cap=1) as eng:
        eng.load_program(prog)
        with pytest.raises(P.ValidationError):
            eng.run_conventional(np.zeros((1, prog.n_sites), np.uint8), np.zeros((1, prog.n_sites)))


def test_conventional_at_20_qubits_with_generated_kernels():
    """A 20-qubit damped brickwork (generated pass kernels, several tiles): device selections
    and weights equal the oracle's Algorithm 1 on the same uniforms (pure numpy restatement)."""
    from paper_2504_16297_b200 import workloads as W
    ctext, _ = W.random_brickwork(20, layers=2, seed=9)
    c = P.attach_noise(P.parse_circuit(ctext), P.parse_noise_model(
        "rule gate=ry qubit=* channel=amplitude_damping(0.2)\nrule gate=cx qubit=* channel=depolarizing(0.05)\n"))
    for t in range(2):
        rng = stream_rng(77, t)
        tr = run_trajectory(c, rng)
        ref = O.run_conventional(c, stream_rng(77, t))
        assert [tuple(p) for p in tr.selections] == ref["selections"]
        assert tr.weight == pytest.approx(ref["weight"], rel=1e-12)
        assert rel(tr.final_state.amplitudes, ref["state"]) <= 1e-12


def test_annihilating_conventional_draw_raises():
    """Clamped draw onto a zero-probability branch -> AnnihilatedStateError, as the reference."""
    c = P.attach_noise(P.parse_circuit("qubits 2\ngate x 0\n"),
                       P.parse_noise_model("channel name=k arity=1\nkraus 1+0i 0+0i 0+0i 0+0i\n"
                                           "kraus 0+0i 0+0i 0+0i 0+0i\nend\n"
                                           "rule gate=x qubit=* channel=k\n", require_cptp=False))
    assert N.TRAJ_ANNIHILATED == 2
    with pytest.raises(P.AnnihilatedStateError):
        run_trajectory(c, np.random.default_rng(0))
