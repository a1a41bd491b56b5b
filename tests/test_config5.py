"""Config 5 (SURVEY 8(e) state sharding) at 34 qubits on one B200: two virtual shards of 33
local qubits (2 x 64 GiB, c64) against the unsharded engine on the same GPU (128 GiB), one
trajectory with 10^6 shots (tools/config5.py does the work).  SURVEY 8(c): no CPU oracle at
this size -- parity is sharded vs unsharded device runs, norm conservation and shot sanity."""

import pytest

pytestmark = pytest.mark.gpu


def test_config5_34q_sharded_equals_unsharded():
    from paper_2504_16297_b200.engine import device_memory
    free, total = device_memory(0)
    if total < 170e9:
        pytest.skip("needs a 180 GB B200")
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tools"))
    import config5
    r = config5.run()
    assert r["status"] == [0, 0]
    assert r["swaps"] >= 1
    assert r["subset_rel_l2"] <= 1e-5                      # c64 tolerance (north_star)
    assert abs(r["norm_total_unsharded"] - 1.0) <= 1e-5
    assert abs(r["norm_total_sharded"] - 1.0) <= 1e-5
    assert r["shots_drawn"] == 1_000_000 and r["sorted_unique"]
    assert r["min_prob_of_sampled"] > 0
