"""GPU check of the circuit-specialised kernels: load time, and state parity vs the generic kernel."""
import os, sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2504_16297_b200 as P
from paper_2504_16297_b200 import workloads
from paper_2504_16297_b200.engine import Engine
from paper_2504_16297_b200.program import selection_matrix

os.makedirs("gpurun_out", exist_ok=True)
for cfg, dtype, nb in [(2, "c128", 4), (3, "c64", 2), (4, "c64", 2)]:
    c = workloads.build(cfg, P.parse_circuit, P.parse_noise_model, P.attach_noise)
    specs = P.presample_probabilistic(c, 50, 10, np.random.default_rng(1))[:nb]
    res = {}
    for mode in ("0", "1"):
        os.environ["PTSBE_CODEGEN"] = mode
        os.environ["PTSBE_CODEGEN_DUMP"] = f"gpurun_out/gen_cfg{cfg}.cu"
        with Engine(c.n_qubits, dtype, batch_cap=nb) as eng:
            t0 = time.perf_counter()
            prog = eng.load(c)
            t1 = time.perf_counter()
            w, st = eng.run(selection_matrix(prog, specs))
            eng.synchronize()
            t2 = time.perf_counter()
            w, st = eng.run(selection_matrix(prog, specs))
            t3 = time.perf_counter()
            res[mode] = [eng.get_state(b).astype(np.complex128) for b in range(nb)]
            print(f"cfg{cfg} {dtype} codegen={mode} info={eng.info()} load {t1-t0:.2f}s run1 {t2-t1:.3f}s run2 {t3-t2:.3f}s", flush=True)
    err = max(np.linalg.norm(a - b) / np.linalg.norm(b) for a, b in zip(res["1"], res["0"]))
    print(f"cfg{cfg}: max rel diff codegen vs generic = {err:.3e}", flush=True)
