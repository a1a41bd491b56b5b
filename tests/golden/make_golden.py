"""Generate golden vectors by running the REFERENCE (``/root/reference/pkg/src/trajsim``).

Run in the build container only (the reference does not exist on the GPU
box):  ``python tests/golden/make_golden.py``.  Writes ``golden.json`` and
``golden.npz`` next to this script; both are committed.  Inputs come from
``paper_2504_16297_b200.workloads`` (plain circuit / noise text) and small
hand-written cases, so the reference's own parser defines the semantics.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))

import trajsim as R  # noqa: E402  (the reference)

from paper_2504_16297_b200 import workloads as W  # noqa: E402

DEMO = Path("/root/reference/pkg/src/trajsim/demos")

SMALL_CASES = {
    # name: (circuit text, noise text or None)
    "rychain_mixture": ((DEMO / "rychain4.circ").read_text(), (DEMO / "rychain_mixture.noise").read_text()),
    "rychain_damped": ((DEMO / "rychain4.circ").read_text(), (DEMO / "rychain_damped.noise").read_text()),
    "teleport_damped": ((DEMO / "teleport5.circ").read_text(),
                        "rule gate=* qubit=* channel=amplitude_damping(0.2)\n"),
    "ghz4_depol": ((DEMO / "ghz4.circ").read_text(), (DEMO / "depol01.noise").read_text()),
    "distill5_custom": ((DEMO / "distill5.circ").read_text(), (DEMO / "custom_example.noise").read_text()),
    "config1": W.ghz_repetition(10),
    "config2": W.surface_code_d3(),
    "brick8": W.random_brickwork(8, layers=4, seed=3, p=0.02),
    "steane1": W.steane_blocks(1, rounds=3, seed=5, p1=0.01, p2=0.01),
}


def build(name):
    ctext, ntext = SMALL_CASES[name]
    c = R.parse_circuit(ctext)
    if ntext is not None:
        c = R.attach_noise(c, R.parse_noise_model(ntext))
    return c


def spec_json(s):
    return {"selections": [list(p) for p in s.selections], "shots": s.shots,
            "joint_prob": s.joint_prob, "tags": s.tags}


def main():
    out = {"numpy": np.__version__, "reference": "/root/reference/pkg/src/trajsim", "cases": {}}
    arrays = {}
    out["mix_seed"] = [[m, s, R.mix_seed(m, s)] for m, s in
                       [(0, 0), (0, 1), (12345, 7), (2**63, 2**32), (42, 99), (7, 2**63)]]
    # PCG64 first uniforms of stream_rng (pins the oracle's PCG64 restatement)
    out["pcg64"] = []
    for m, s in [(0, 0), (3, 5), (2**40, 17)]:
        g = R.stream_rng(m, s)
        st = g.bit_generator.state["state"]
        out["pcg64"].append({"master": m, "stream": s, "state": str(st["state"]), "inc": str(st["inc"]),
                             "uniforms": [float(x) for x in g.random(8)]})
    for name, (ctext, ntext) in SMALL_CASES.items():
        c = build(name)
        case = {"circuit": ctext, "noise": ntext, "n_qubits": c.n_qubits,
                "circuit_sha256": R.circuit_hash(c), "sites_sha256": R.circuit.sites_hash(c),
                "n_ops": len(c.ops), "n_sites": len(c.sites),
                "moments": list(c.moments),
                "sites": [[s.site_id, s.position, s.moment, list(s.targets), s.channel_id] for s in c.sites]}
        table = R.site_outcome_probs(c)
        all_mix = all(e.is_mixture for e in table)
        case["site_probs"] = [[float(x) for x in e.probs] for e in table]
        # PTS strategies (host, must be bit-exact)
        pts = {}
        raw = []
        specs = R.presample_probabilistic(c, 200, 1000, np.random.default_rng(11), raw_sink=raw)
        pts["probabilistic"] = [spec_json(s) for s in specs]
        pts["probabilistic_raw"] = [[list(p) for p in r] for r in raw[:50]]
        if c.n_qubits >= 2 and len(c.sites):
            flt = R.SiteFilter(qubits=frozenset({0, 1}))
            pts["filtered"] = [spec_json(s) for s in
                               R.presample_probabilistic(c, 100, 10, np.random.default_rng(5), site_filter=flt)]
        if all_mix and len(c.sites):
            band = R.presample_band(c, 1e-4, 0.5, 300, 7, np.random.default_rng(2))
            pts["band"] = [spec_json(s) for s in band]
            pts["proportional"] = [spec_json(s) for s in R.reallocate_proportional(specs, 12345)]
            cut = 1e-3 if c.n_qubits < 12 else 1e-5
            pts["cutoff"] = [spec_json(s) for s in R.enumerate_cutoff(c, cut, 50)]
            case["cutoff_value"] = cut
        case["pts"] = pts
        # prepared states for the first specs + reference sampling
        preps = []
        use = specs[:12]
        for i, s in enumerate(use):
            try:
                st, w = R.prepare_state(c, s)
            except R.AnnihilatedStateError as exc:
                preps.append({"selections": [list(p) for p in s.selections], "annihilated": str(exc)})
                continue
            key = f"{name}__amp{i}"
            arrays[key] = st.amplitudes
            batch = R.sample_shots(st, 5000, R.stream_rng(9, i))
            preps.append({"selections": [list(p) for p in s.selections], "weight": w, "amps": key,
                          "sample_seed": [9, i], "sample_m": 5000, "counts": batch.counts})
        case["prepared"] = preps
        # a full execute_all dataset (records + manifest core)
        ds = R.execute_all(c, use, parallelism=1, master_seed=21)
        case["dataset"] = {"master_seed": 21,
                           "records": [[r.trajectory_id, r.bitstring, r.count] for r in ds.records],
                           "manifest_core": R.manifest_core(ds.manifest)}
        out["cases"][name] = case
        print(name, c.n_qubits, len(c.ops), len(c.sites), len(specs), file=sys.stderr)
    # a larger state for sampler parity: bench20 noise-free (checksums only)
    c20 = R.parse_circuit((DEMO / "bench20.circ").read_text())
    st, _w = R.prepare_state(c20, R.TrajectorySpec((), 0))
    probs = st.probabilities()
    out["bench20"] = {"circuit": (DEMO / "bench20.circ").read_text(),
                      "prob_sum_by_1024": [float(x) for x in probs.reshape(-1, 1024).sum(axis=1)],
                      "amps_head": [[float(a.real), float(a.imag)] for a in st.amplitudes[:64]],
                      "counts_m1000_seed00": R.sample_shots(st, 1000, R.stream_rng(0, 0)).counts}
    (HERE / "golden.json").write_text(json.dumps(out, indent=1, sort_keys=True))
    np.savez_compressed(HERE / "golden.npz", **arrays)
    print("wrote", HERE / "golden.json", HERE / "golden.npz", file=sys.stderr)


if __name__ == "__main__":
    main()
