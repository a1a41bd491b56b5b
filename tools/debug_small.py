import numpy as np, sys
sys.path.insert(0, '.')
import paper_2504_16297_b200 as P
from paper_2504_16297_b200.engine import Engine
for dtype in ("c128", "c64"):
    for text in ["qubits 1\ngate x 0\n", "qubits 2\ngate h 0\ngate cx 0 1\n", "qubits 4\ngate h 0\ngate h 3\n"]:
        c = P.parse_circuit(text)
        with Engine(c.n_qubits, dtype, 1) as eng:
            prog = eng.load(c)
            print(dtype, repr(text), "passes", [(p.qubits, p.low_bits, p.ops) for p in prog.passes], eng.info())
            w, s = eng.run(np.zeros((1, 0), np.uint8))
            print("  w,s", w, s, "state", np.round(eng.get_state(0), 4))
            a = np.arange(1 << c.n_qubits).astype(np.complex128)
            eng.set_state(0, a)
            print("  roundtrip", np.array_equal(eng.get_state(0), a.astype(eng.np_dtype)))
