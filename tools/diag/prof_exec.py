import cProfile, pstats, sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2504_16297_b200 as P
from paper_2504_16297_b200 import workloads
from paper_2504_16297_b200.execute import execute_all, stream_rng, run_specs
c = workloads.build(3, P.parse_circuit, P.parse_noise_model, P.attach_noise)
specs = P.presample_probabilistic(c, 200, 10000, stream_rng(1, 2**63))
run_specs(c, specs, 1, dtype="c64", rng="philox")
specs = P.presample_probabilistic(c, 2000, 10000, stream_rng(3, 2**63))
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
ds = execute_all(c, specs, master_seed=3, dtype="c64", rng="philox")
pr.disable()
print("execute_all", time.perf_counter() - t0, len(specs))
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
