"""Fusion planner: every plan is a legal reordering of the reference's op loop.

The planned order (pass by pass) is executed with the CPU oracle and compared
with the reference's sequential order (execute.py:85-97); per pass the targets
must lie in the pass's qubit set and qubits 0..c-1 must be in it.
"""

import numpy as np
import pytest

import paper_2504_16297_b200 as P
from paper_2504_16297_b200 import workloads as W
from paper_2504_16297_b200.program import KIND_GATE, compile_circuit, plan_passes, selection_matrix
from oracle import engine as O


def _run_stream(c, prog, order, sel):
    psi = O.zero_state(c.n_qubits)
    w = 1.0
    for i in order:
        so = prog.stream[i]
        if so.kind == KIND_GATE:
            m = prog.mats[so.ref][: 1 << len(so.targets), : 1 << len(so.targets)]
            psi = O.apply_local(psi, m, so.targets, c.n_qubits)
            continue
        ch = prog.chans[int(prog.site_chan[so.ref])]
        k = int(sel[so.ref])
        if (ch["identity_mask"] >> k) & 1:
            continue
        d = 1 << len(so.targets)
        m = prog.mats[ch["mat_base"] + k][:d, :d]
        psi = O.apply_local(psi, m, so.targets, c.n_qubits)
        if ch["general"]:
            r = float(np.sum(np.abs(psi) ** 2))
            psi = psi / np.sqrt(r)
            w *= r
    return psi, w


@pytest.mark.parametrize("tile_bits,low_bits", [(4, 2), (5, 3), (6, 4)])
@pytest.mark.parametrize("name", ["brick8", "steane1", "teleport_damped", "distill5_custom"])
def test_plan_is_legal_reordering(golden, name, tile_bits, low_bits):
    from conftest import build_case
    c = build_case(golden["cases"][name])
    prog = compile_circuit(c, "c128", tile_bits=tile_bits, low_bits=low_bits)
    order = [i for p in prog.passes for i in p.ops]
    assert sorted(order) == list(range(len(prog.stream)))
    perm = prog.perm
    assert sorted(perm) == list(range(c.n_qubits))
    for p in prog.passes:
        assert len(p.qubits) == min(c.n_qubits, tile_bits)
        assert tuple(range(p.low_bits)) == p.qubits[: p.low_bits]
        for i in p.ops:
            assert {perm[q] for q in prog.stream[i].targets} <= set(p.qubits)
    rng = np.random.default_rng(1)
    specs = P.presample_probabilistic(c, 40, 1, rng)
    sel = selection_matrix(prog, specs)
    for b, spec in enumerate(specs[:8]):
        try:
            ref_psi, ref_w = O.prepare(c, spec.selections)
        except O.Annihilated:
            continue
        psi, w = _run_stream(c, prog, order, sel[b])
        assert np.linalg.norm(psi - ref_psi) <= 1e-12
        assert w == pytest.approx(ref_w, rel=1e-12)


@pytest.mark.parametrize("name", ["brick8", "steane1", "config2"])
def test_native_planner_matches_python_planner(golden, name):
    from conftest import build_case
    from paper_2504_16297_b200.program import lower, plan_native
    c = build_case(golden["cases"][name])
    prog = lower(c)
    for L, lowb in [(5, 3), (6, 4), (12, 4)]:
        py = plan_passes(c.n_qubits, prog.stream, L, lowb)
        perm, nat = plan_native(c.n_qubits, prog.stream, L, lowb, search_iters=0)
        assert perm == list(range(c.n_qubits))
        assert [(p.qubits, p.low_bits, p.ops) for p in py] == [(p.qubits, p.low_bits, p.ops) for p in nat]


def test_layout_search_reduces_passes_config4():
    from paper_2504_16297_b200.program import lower, plan_native
    c = W.build(4, P.parse_circuit, P.parse_noise_model, P.attach_noise)
    prog = lower(c)
    _, base = plan_native(28, prog.stream, 12, 4, search_iters=0)
    perm, best = plan_native(28, prog.stream, 12, 4, search_iters=3000)
    assert len(best) <= len(base) * 0.6
    # every op's physical targets inside its pass; the reordering is legal (same rule as Python)
    for p in best:
        for i in p.ops:
            assert {perm[q] for q in prog.stream[i].targets} <= set(p.qubits)


def test_plan_counts_for_configs():
    c = W.build(4, P.parse_circuit, P.parse_noise_model, P.attach_noise)
    prog = compile_circuit(c, "c64")
    assert prog.g_ref == len(c.ops) + len(c.sites)
    assert prog.n_passes < prog.g_ref / 10          # >= 10x fewer HBM passes than the reference
    small = W.build(1, P.parse_circuit, P.parse_noise_model, P.attach_noise)
    assert compile_circuit(small, "c128").n_passes == 1   # whole 10 q circuit in one smem pass


def test_identity_gates_dropped_and_identity_outcomes_masked():
    c = P.attach_noise(P.parse_circuit("qubits 2\ngate i 0\ngate h 1\n"),
                       P.parse_noise_model("rule gate=* qubit=* channel=depolarizing(0.1)\n"))
    prog = compile_circuit(c, "c128")
    assert [s.kind for s in prog.stream] == [1, 0, 1]    # 'i' gate removed, both sites kept
    assert all(ch["identity_mask"] == 1 for ch in prog.chans)


def _conv_case(name):
    import json
    from conftest import GOLDEN, build_case
    return build_case(json.loads((GOLDEN / "golden_conv.json").read_text())["cases"][name])


@pytest.mark.parametrize("tile_bits,low_bits", [(4, 2), (6, 3), (11, 3), (12, 4)])
@pytest.mark.parametrize("name", ["teleport_damped", "brick8_mixed", "ghz10_damped", "brick11_mixed"])
def test_conventional_plan_opens_a_pass_at_every_general_site(name, tile_bits, low_bits):
    """Planning for conventional trajectories (decision sites, ptsbe_plan bit 2): every
    general-channel site is the first op of its pass -- its outcome is chosen from the state at
    the pass boundary -- and the plan is still a legal reordering of the reference's loop."""
    c = _conv_case(name)
    prog = compile_circuit(c, "c128", tile_bits=tile_bits, low_bits=low_bits, decide_general=True)
    order = [i for p in prog.passes for i in p.ops]
    assert sorted(order) == list(range(len(prog.stream)))
    n_general = sum(1 for so in prog.stream if so.general)
    assert n_general > 0
    opened = [p.ops[0] for p in prog.passes if prog.stream[p.ops[0]].general]
    assert sum(1 for p in prog.passes for i in p.ops if prog.stream[i].general) == len(opened) == n_general
    # ops a decision site may overtake or be overtaken by act on other qubits and are unitary
    pos = {i: k for k, i in enumerate(order)}
    for i, so in enumerate(prog.stream):
        if not so.general:
            continue
        for j, other in enumerate(prog.stream):
            moved = (j < i and pos[j] > pos[i]) or (j > i and pos[j] < pos[i])
            if moved:
                assert not set(other.targets) & set(so.targets)
                assert not other.general
    # the planned order gives the reference's state for sampled outcomes
    rng = np.random.default_rng(3)
    specs = P.presample_probabilistic(c, 30, 1, rng)
    sel = selection_matrix(prog, specs)
    for b, spec in enumerate(specs[:4]):
        try:
            ref_psi, ref_w = O.prepare(c, spec.selections)
        except O.Annihilated:
            continue
        psi, w = _run_stream(c, prog, order, sel[b])
        assert np.linalg.norm(psi - ref_psi) <= 1e-12
        assert w == pytest.approx(ref_w, rel=1e-12)


def test_conventional_plan_small_state_cuts_single_tile():
    """n <= tile bits: one tile per pass, a new pass before each general site (not the first op)."""
    c = _conv_case("teleport_damped")
    prog = compile_circuit(c, "c128", decide_general=True)
    n_general = sum(1 for so in prog.stream if so.general)
    first_general = prog.stream[0].general
    assert prog.n_passes == n_general + (0 if first_general else 1)
    assert all(len(p.qubits) == c.n_qubits for p in prog.passes)
