"""Diagnostic: per-pass coset-norm conservation of the config-4 plan on a random state."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2504_16297_b200 as P
from paper_2504_16297_b200 import workloads
from paper_2504_16297_b200.engine import Engine
from paper_2504_16297_b200.program import compile_circuit
from test_config4_parity import hit_selections, logical_qubits, random_state, oracle_items, coset_rows, check_pass

dtype = sys.argv[1] if len(sys.argv) > 1 else "c64"
c = workloads.build(4, P.parse_circuit, P.parse_noise_model, P.attach_noise)
rng = np.random.default_rng(4)
prog = compile_circuit(c, dtype)
selections, sel = hit_selections(c, prog, rng)
psi = random_state(28, dtype)
n = 28

def coset_norms(st, qs):
    t = np.abs(st.astype(np.complex128)) ** 2
    t = t.reshape((2,) * n)
    axes_q = [n - 1 - q for q in qs]
    rest = [a for a in range(n) if a not in axes_q]
    return np.transpose(t, rest + axes_q).reshape(1 << len(rest), -1).sum(axis=1)

with Engine(28, dtype, batch_cap=3) as eng:
    eng.load_program(prog)
    for p in range(prog.n_passes):
        print(p, eng.pass_info(p), flush=True)
    for b in range(3):
        eng.set_state(b, psi)
    prev = [psi] * 3
    for p in range(prog.n_passes):
        eng.run_range(sel, p, p + 1, continue_=True)
        cur = [eng.get_state(b) for b in range(3)]
        qs = logical_qubits(prog, p)
        for b in range(3):
            a0 = coset_norms(prev[b], qs); a1 = coset_norms(cur[b], qs)
            d = np.abs(a1 - a0)
            bad = np.flatnonzero(d > 1e-6 * a0.mean() * 100)
            print(f"pass {p} b {b}: total {a0.sum():.6f} -> {a1.sum():.6f}; bad cosets {bad.size}"
                  f" first {bad[:8].tolist()} ratio {(a1[bad[:4]] / a0[bad[:4]]).tolist()}", flush=True)
        prev = cur
