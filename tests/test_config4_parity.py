"""Config 4 (the bench program, 28 q) against the oracle, pass by pass, in c64 and c128.

The bench's own generated pass kernels (``ptsbe_pass_<p>``, every pass of the
plan ``compile_circuit`` makes for config 4 -- 4-bit and 5-bit register
phases, fast bodies and the out-of-line slow variants for sites with a
non-default outcome, the last pass) are run one pass at a time with
``ptsbe_run_range`` on 28-qubit states and compared with the oracle applying
that pass's operators (reference order, ``execute.py:85-97``) to the same
input.  A full 28-q oracle pass is minutes of numpy per pass, so the check is
made on cosets: the operators of a pass act inside its tile qubit set Q, hence
independently on every coset of Q (a fixed pattern of the other 16-17
qubits), and ``oracle.apply_on_cosets`` applied to a few hundred random cosets
gives exactly the full-state result on those amplitudes.

Tolerances: north_star's norm-wise 1e-5 (c64) / 1e-12 (c128).  A single pass
run alone is compared up to one global phase (fitted over all sampled cosets):
the generated kernels fold the program's accumulated global phase into pass 0
(codegen.h), so a pass on its own applies its operators times a unit constant.
The complete program carries no such freedom: the pass-by-pass chain from
|0...0> equals ``run_batch``'s bench path (shared trunk, fused sampler sums)
bit for bit, and the PCG64 verification-mode shots of those 28-q states equal
the reference sampler's on the downloaded amplitudes.
"""

import numpy as np
import pytest

import paper_2504_16297_b200 as P
from paper_2504_16297_b200 import _native as N
from paper_2504_16297_b200 import workloads
from paper_2504_16297_b200.engine import Engine, pcg64_state_words
from paper_2504_16297_b200.execute import mix_seed
from paper_2504_16297_b200.program import KIND_GATE, compile_circuit, selection_matrix
from oracle import engine as O

pytestmark = pytest.mark.gpu

TOL = {"c128": 1e-12, "c64": 1e-5}
COSETS = {"c128": 256, "c64": 512}


@pytest.fixture(scope="module")
def config4():
    return workloads.build(4, P.parse_circuit, P.parse_noise_model, P.attach_noise)


def logical_qubits(prog, p):
    """Tile qubit set of pass p in LOGICAL qubits (pass masks are physical)."""
    perm = list(range(prog.n_qubits)) if prog.perm is None else list(prog.perm)
    phys = set(prog.passes[p].qubits)
    return sorted(q for q in range(prog.n_qubits) if perm[q] in phys)


def oracle_items(circuit, prog, p, selections):
    """The oracle's (matrix, targets) for the ops of pass p, in the pass's order."""
    items = []
    for i in prog.passes[p].ops:
        so = prog.stream[i]
        if so.kind == KIND_GATE:
            items.append(O.gate_item(circuit, so.pos))
        else:
            mat, targets, general = O.site_item(circuit, so.ref, selections)
            assert not general
            items.append((mat, targets))
    return items


def hit_selections(circuit, prog, rng):
    """Three trajectories: no error; one error per pass; up to three per pass at spread sites
    (different slow-variant segments).  Returns (selections, (B, S) outcome table)."""
    sels = [[], [], []]
    for plan in prog.passes:
        sites = [prog.stream[i].ref for i in plan.ops if prog.stream[i].kind != KIND_GATE]
        if not sites:
            continue
        picks = {1: [sites[len(sites) // 2]], 2: sorted({sites[0], sites[len(sites) // 3], sites[-1]})}
        for b, ss in picks.items():
            for s in ss:
                n_out = len(circuit.channels[circuit.site(s).channel_id].kraus_ops)
                sels[b].append((s, int(rng.integers(1, n_out))))
    selections = [tuple(sorted(s)) for s in sels]
    specs = [P.TrajectorySpec(s, 0) for s in selections]
    return selections, selection_matrix(prog, specs)


def coset_rows(n, qubits, count, rng):
    """(count, 2^|Q|) logical indices of `count` random cosets of Q (always incl. the first/last)."""
    rest = [q for q in range(n) if q not in qubits]
    pats = rng.choice(1 << len(rest), size=count, replace=False)
    pats[0], pats[-1] = 0, (1 << len(rest)) - 1
    lo = O.scatter_bits(np.arange(1 << len(qubits)), qubits)
    hi = O.scatter_bits(pats, rest)
    return hi[:, None] | lo[None, :]


def check_pass(prev, cur, items, qubits, idx, tol, phase_free=True):
    ref = O.apply_on_cosets(prev[idx].astype(np.complex128), items, qubits)
    dev = cur[idx].astype(np.complex128)
    if phase_free:
        ov = np.vdot(ref, dev)
        assert abs(ov) > 0
        dev = dev * (np.conj(ov) / abs(ov))
    err = float(np.linalg.norm(dev - ref) / max(np.linalg.norm(ref), 1e-300))
    assert err <= tol, err
    return err


def coset_norms(state, qubits):
    """Norm^2 of every coset of the qubit set (float64)."""
    n = state.size.bit_length() - 1
    t = (np.abs(state.astype(np.complex128)) ** 2).reshape((2,) * n)
    axes_q = [n - 1 - q for q in qubits]
    rest = [a for a in range(n) if a not in axes_q]
    return np.transpose(t, rest + axes_q).reshape(1 << len(rest), -1).sum(axis=1)


def random_state(n, dtype, seed=0):
    rng = np.random.default_rng(seed)
    psi = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    psi /= np.linalg.norm(psi)
    return psi.astype(np.complex64 if dtype == "c64" else np.complex128)


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_every_bench_pass_against_oracle_random_input(config4, dtype):
    """Each generated pass of the config-4 plan on a random 28-q state: three trajectories
    (fast path, one slow site, several slow segments) against the oracle on sampled cosets."""
    c = config4
    rng = np.random.default_rng(4)
    prog = compile_circuit(c, dtype)
    selections, sel = hit_selections(c, prog, rng)
    psi = random_state(c.n_qubits, dtype)
    with Engine(c.n_qubits, dtype, batch_cap=3) as eng:
        eng.load_program(prog)
        assert eng.info()["codegen"] == 1
        widths = {eng.pass_info(p)["gb"] for p in range(prog.n_passes)}
        if dtype == "c64":
            assert widths == {4, 5}        # both register-phase widths of the plan are exercised
        for b in range(3):
            eng.set_state(b, psi)
        prev = [psi] * 3
        del psi
        for p in range(prog.n_passes):
            eng.run_range(sel, p, p + 1, continue_=True)
            cur = [eng.get_state(b) for b in range(3)]
            qs = logical_qubits(prog, p)
            idx = coset_rows(c.n_qubits, qs, COSETS[dtype], rng)
            for b in range(3):
                check_pass(prev[b], cur[b], oracle_items(c, prog, p, selections[b]), qs, idx, TOL[dtype])
            # unitary pass: every state keeps its norm (exact 2^-62 fixed-point sum on device)
            n2 = eng.norm_totals(3).astype(np.float64) / 2.0 ** 62
            assert np.all(np.abs(n2 - 1.0) <= (1e-5 if dtype == "c64" else 1e-12)), n2
            if dtype == "c64" and eng.pass_info(p)["gb"] == 4:
                # every coset of Q keeps its norm (the pass is unitary inside each coset): a
                # full-state check of the tile addressing of the 4-bit (256-thread) passes
                a0, a1 = coset_norms(prev[2], qs), coset_norms(cur[2], qs)
                assert np.max(np.abs(a1 - a0)) <= 1e-5 * max(float(a0.max()), 1e-30)
            prev = cur


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_config4_trajectories_chain_equals_bench_path_and_oracle(config4, dtype):
    """Two PTS-sampled config-4 trajectories from |0...0>: pass-by-pass chain checked against the
    oracle on cosets, final states bit-identical to run_batch (the bench path), and in c128
    the PCG64 verification-mode shots equal the reference sampler on those 28-q states."""
    c = config4
    rng = np.random.default_rng(5)
    specs = [s for s in P.presample_probabilistic(c, 40, 10_000, np.random.default_rng(3)) if s.selections][:2]
    assert len(specs) == 2
    prog = compile_circuit(c, dtype)
    sel = selection_matrix(prog, specs)
    with Engine(c.n_qubits, dtype, batch_cap=2) as eng:
        eng.load_program(prog)
        w, st = eng.run(sel)                      # the bench path: shared trunk + fused sums
        assert list(st) == [0, 0] and np.all(w == 1.0)
        bench = [eng.get_state(b) for b in range(2)]
        prev = None
        for p in range(prog.n_passes):
            eng.run_range(sel, p, p + 1)          # pass 0 starts from |0...0>
            cur = [eng.get_state(b) for b in range(2)]
            if prev is not None:
                qs = logical_qubits(prog, p)
                idx = coset_rows(c.n_qubits, qs, COSETS[dtype], rng)
                for b in range(2):
                    check_pass(prev[b], cur[b], oracle_items(c, prog, p, specs[b].selections), qs, idx, TOL[dtype])
            prev = cur
        for b in range(2):
            assert np.array_equal(prev[b], bench[b])
        del bench, prev, cur
        if dtype == "c128":
            words = np.concatenate([pcg64_state_words(mix_seed(2024, t)) for t in range(2)])
            out = eng.sample([10_000, 10_000], N.RNG_PCG64, rng_state=words)
            for b in range(2):
                psi = eng.get_state(b)
                rng_b = np.random.Generator(np.random.PCG64(mix_seed(2024, b)))
                assert out.counts_dict(b, 28) == O.sample(psi, 10_000, rng_b, 28)
