import sys; sys.path.insert(0, ".")
import numpy as np
from scipy import stats
import paper_2504_16297_b200 as P
from paper_2504_16297_b200 import workloads
from paper_2504_16297_b200.sharded import plan_sharded, sharded_selection, VirtualShards
from paper_2504_16297_b200.engine import Engine
from paper_2504_16297_b200 import _native as N
from paper_2504_16297_b200.execute import mix_seed
from oracle import engine as O
text, noise = workloads.random_brickwork(12, layers=4, seed=5, p=0.05)
c = P.attach_noise(P.parse_circuit(text), P.parse_noise_model(noise))
specs = P.presample_probabilistic(c, 60, 50_000, np.random.default_rng(6))[:3]
ref, _ = O.prepare(c, specs[0].selections); probs = np.abs(ref) ** 2
top = np.argsort(probs)[::-1][:10]
def pv(idx, cnt, m):
    obs = np.array([cnt[idx == t].sum() for t in top], dtype=float); exp = probs[top] * m
    return stats.chisquare(np.append(obs, m - obs.sum()), np.append(exp, m - exp.sum())).pvalue
for k in (0, 1, 2):
    ps = []
    if k == 0:
        with Engine(12, "c128", 1) as e:
            e.set_state(0, ref)
            for r in range(40):
                out = e.sample([50000], N.RNG_PHILOX, rng_state=np.array([mix_seed(99, r)], dtype=np.uint64))
                ps.append(pv(out.indices, out.counts, 50000))
    else:
        plan = plan_sharded(c, k, dtype="c128", tile_bits=6, low_bits=3)
        vs = VirtualShards(plan, "c128", batch_cap=1)
        vs.run(sharded_selection(plan, specs[:1]))
        for r in range(40):
            idx, cnt = vs.sample([50000], [mix_seed(99, r)])[0]
            ps.append(pv(idx, cnt, 50000))
        vs.close()
    ps = np.array(ps)
    print(k, "min p", ps.min().round(4), "frac<0.05", (ps < 0.05).mean(), "KS-uniform p", stats.kstest(ps, "uniform").pvalue.round(4), flush=True)
