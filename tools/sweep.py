"""Config-4 pass-time sweep over tile bits / phase bits (c64): ms per batch of B trajectories."""
import os, sys, time, json
sys.path.insert(0, ".")
import numpy as np
import paper_2504_16297_b200 as P
from paper_2504_16297_b200 import workloads
from paper_2504_16297_b200.engine import Engine
from paper_2504_16297_b200.program import compile_circuit, selection_matrix
c = workloads.build(4, P.parse_circuit, P.parse_noise_model, P.attach_noise)
specs = P.presample_probabilistic(c, 60, 10000, np.random.default_rng(5))[:8]
res = []
for L, gb in [(12, 4), (12, 5), (13, 4), (13, 5), (11, 4)]:
    os.environ["PTSBE_PHASE_BITS"] = str(gb)
    prog = compile_circuit(c, "c64", tile_bits=L)
    with Engine(28, "c64", batch_cap=8) as eng:
        eng.load_program(prog)
        sel = selection_matrix(prog, specs)
        eng.run(sel); eng.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            eng.run(sel)
        eng.synchronize()
        ms = (time.perf_counter() - t0) / 3 * 1e3
        r = dict(L=L, gb=gb, passes=prog.n_passes, info=eng.info()["n_phases"], ms=round(ms, 2),
                 gbps=round(prog.n_passes * 2 * 8 * (1 << 28) * 8 / (ms / 1e3) / 1e9, 1))
        print(json.dumps(r), flush=True)
