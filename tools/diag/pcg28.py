"""Where do device PCG64 shots and numpy's sample_shots differ on the 28-q config-4 states?

Run on the GPU box: python tools/diag/pcg28.py > gpurun_out/pcg28.txt
Prepares the two trajectories of tests/test_config4_parity.py (c128), samples 10^4 PCG64
shots on device, replays numpy's sample_shots on the downloaded amplitudes, and for every
shot whose index differs prints the uniform, both CDFs around it and an extended-precision
reference."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2504_16297_b200 as P  # noqa: E402
from paper_2504_16297_b200 import _native as N, workloads  # noqa: E402
from paper_2504_16297_b200.engine import Engine, pcg64_state_words  # noqa: E402
from paper_2504_16297_b200.execute import mix_seed  # noqa: E402
from paper_2504_16297_b200.program import compile_circuit, selection_matrix  # noqa: E402

c = workloads.build(4, P.parse_circuit, P.parse_noise_model, P.attach_noise)
specs = [s for s in P.presample_probabilistic(c, 40, 10_000, np.random.default_rng(3)) if s.selections][:2]
prog = compile_circuit(c, "c128")
m = 10_000
with Engine(c.n_qubits, "c128", batch_cap=2) as eng:
    eng.load_program(prog)
    eng.run(selection_matrix(prog, specs))
    words = np.concatenate([pcg64_state_words(mix_seed(2024, t)) for t in range(2)])
    out = eng.sample([m, m], N.RNG_PCG64, rng_state=words)
    for b in range(2):
        psi = eng.get_state(b)
        u = np.random.Generator(np.random.PCG64(mix_seed(2024, b))).random(m)
        p = np.abs(psi) ** 2
        cum = np.cumsum(p)
        cdf = cum / cum[-1]
        idx_np = np.clip(np.searchsorted(cdf, u, side="right"), 0, p.size - 1)
        # device emulation: q = rn(fl(fl(x^2)+fl(y^2)) * 2^62), integer prefix, target = floor(K*T/2^53)
        pd = psi.real * psi.real + psi.imag * psi.imag
        q = np.rint(pd * 2.0 ** 62).astype(np.uint64)
        Q = np.cumsum(q)
        T = int(Q[-1])
        K = (u * 2.0 ** 53).astype(np.uint64)
        tgt = np.array([(int(k) * T) >> 53 for k in K], dtype=np.uint64)
        idx_em = np.searchsorted(Q, tgt, side="right")
        lo, hi = int(out.offsets[b]), int(out.offsets[b + 1])
        dev = np.repeat(out.indices[lo:hi].astype(np.int64), out.counts[lo:hi])
        print(f"traj {b}: nonzero p {np.count_nonzero(p)}, support max p {p.max():.3e}, sum-1 {cum[-1]-1:.3e}, "
              f"device==emulation {np.array_equal(np.sort(idx_em), dev)}, numpy==emulation "
              f"{np.array_equal(np.sort(idx_np), np.sort(idx_em))}")
        bad = np.flatnonzero(idx_np != idx_em)
        cl = np.cumsum(p.astype(np.longdouble))
        for i in bad[:10]:
            j0, j1 = sorted((int(idx_np[i]), int(idx_em[i])))
            print(f"  shot {i}: u={u[i]!r} numpy idx {idx_np[i]} device idx {idx_em[i]}")
            for j in range(max(0, j0 - 2), min(p.size, j1 + 2)):
                print(f"    j={j} p={p[j]!r} pd={pd[j]!r} cdf_np={cdf[j]!r} Q/T={Q[j] / T!r} "
                      f"ext={(cl[j] / cl[-1])!r} np<=u {cdf[j] <= u[i]} dev<=u {Q[j] <= tgt[i]}")
