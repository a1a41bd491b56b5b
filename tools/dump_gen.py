import os, sys
sys.path.insert(0, ".")
import numpy as np
import paper_2504_16297_b200 as P
from paper_2504_16297_b200 import workloads
from paper_2504_16297_b200.engine import Engine
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
dtype = sys.argv[2] if len(sys.argv) > 2 else "c64"
os.environ["PTSBE_CODEGEN"] = "1"
os.environ["PTSBE_CODEGEN_DUMP"] = f"gpurun_out/gen_cfg{cfg}_{dtype}.cu"
c = workloads.build(cfg, P.parse_circuit, P.parse_noise_model, P.attach_noise)
with Engine(c.n_qubits, dtype, batch_cap=1) as eng:
    prog = eng.load(c)
    print(eng.info(), prog.perm)
