"""Golden vectors for the boundary's secondary entry points, made by running the REFERENCE.

Covers what ``make_golden.py`` does not:
  * conventional Algorithm-1 trajectories (``trajectory.py:40-70`` run_trajectory,
    ``:73-106`` sample_conventional, both its dense-ensemble path (n <= 8,
    ``:138-219``) and its per-trajectory path) -- selections, weights, final
    amplitudes, datasets;
  * ``execute_trajectory`` (``execute.py:101-111``), ``execute_naive`` (``:114-127``),
    ``throughput_report`` / ``write_throughput_csv`` (``:320-349``, deterministic
    columns only);
  * ``kraus_outcome_probability`` on prepared (non-trivial) states (``statevector.py:129-133``);
  * the CLI's ``run`` / ``bench`` outputs (``cli.py:146-219``): records.jsonl bytes,
    manifest core, uniqueness.csv, throughput.csv's deterministic columns.

Build container only (``/root/reference`` is not on the GPU box):
``python tests/golden/make_golden_conv.py`` -> ``golden_conv.json`` + ``golden_conv.npz``.
"""

from __future__ import annotations

import json
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))

import trajsim as R  # noqa: E402  (the reference)
import trajsim.trajectory as RT  # noqa: E402
from trajsim.cli import main as ref_cli  # noqa: E402

from paper_2504_16297_b200 import workloads as W  # noqa: E402

DEMO = Path("/root/reference/pkg/src/trajsim/demos")
DAMP = "rule gate=* qubit=* channel=amplitude_damping({p})\n"


def ghz_damped(n, p):
    ctext, _ = W.ghz_repetition(n)
    return ctext, DAMP.format(p=p)


def mixed_noise(p):
    # general (amplitude damping) on h, unitary mixture (depolarizing) on cx
    return (f"rule gate=h qubit=* channel=amplitude_damping({p})\n"
            f"rule gate=ry qubit=* channel=amplitude_damping({p})\n"
            f"rule gate=cx qubit=* channel=depolarizing({p})\n")


CASES = {
    # dense-ensemble path (n <= 8)
    "teleport_damped": ((DEMO / "teleport5.circ").read_text(), DAMP.format(p=0.2)),
    "ghz4_depol": ((DEMO / "ghz4.circ").read_text(), (DEMO / "depol01.noise").read_text()),
    "rychain_damped": ((DEMO / "rychain4.circ").read_text(), (DEMO / "rychain_damped.noise").read_text()),
    "brick8_mixed": (W.random_brickwork(8, layers=3, seed=4)[0], mixed_noise(0.05)),
    # per-trajectory path (n > 8)
    "ghz10_damped": ghz_damped(10, 0.05),
    "config1": W.ghz_repetition(10),
    "brick11_mixed": (W.random_brickwork(11, layers=3, seed=6)[0], mixed_noise(0.03)),
}


def build(ctext, ntext):
    c = R.parse_circuit(ctext)
    if ntext is not None:
        c = R.attach_noise(c, R.parse_noise_model(ntext))
    return c


def dataset_json(ds):
    return {"records": [[r.trajectory_id, r.bitstring, r.count] for r in ds.records],
            "manifest_core": R.manifest_core(ds.manifest)}


def main():
    out = {"numpy": np.__version__, "reference": "/root/reference/pkg/src/trajsim", "cases": {}}
    arrays = {}
    for name, (ctext, ntext) in CASES.items():
        c = build(ctext, ntext)
        case = {"circuit": ctext, "noise": ntext, "n_qubits": c.n_qubits, "n_sites": len(c.sites)}
        # run_trajectory on per-trajectory streams
        runs = []
        for t in range(6):
            rng = R.stream_rng(31, t)
            tr = RT.run_trajectory(c, rng)
            key = f"{name}__run{t}"
            arrays[key] = tr.final_state.amplitudes
            runs.append({"seed": [31, t], "selections": [list(p) for p in tr.selections],
                         "weight": tr.weight, "amps": key,
                         "next_uniform": float(rng.random())})
        case["run_trajectory"] = runs
        # sample_conventional datasets
        conv = {}
        for n_traj, m, seed in [(40, 1, 3), (12, 200, 8)]:
            ds = RT.sample_conventional(c, n_traj, m, master_seed=seed)
            conv[f"{n_traj}x{m}_s{seed}"] = dict(n_traj=n_traj, shots=m, master_seed=seed, **dataset_json(ds))
        case["sample_conventional"] = conv
        # execute_trajectory / execute_naive on PTS specs
        specs = R.presample_probabilistic(c, 60, 300, np.random.default_rng(2))[:4]
        et = []
        for i, s in enumerate(specs):
            try:
                res = R.execute_trajectory(c, s, R.stream_rng(13, i))
            except R.AnnihilatedStateError as exc:
                et.append({"selections": [list(p) for p in s.selections], "annihilated": str(exc)})
                continue
            nb, _dt = R.execute_naive(c, s, 25, R.stream_rng(17, i))
            et.append({"selections": [list(p) for p in s.selections], "shots": s.shots,
                       "weight": res.realized_weight, "counts": res.batch.counts,
                       "naive_counts": nb.counts, "naive_total": nb.total})
        case["execute_trajectory"] = et
        # kraus_outcome_probability on a prepared state, every Kraus op of every channel
        st, _w = R.prepare_state(c, R.TrajectorySpec((), 0))
        kop = []
        for site in c.sites[:6]:
            ch = c.channels[site.channel_id]
            kop.append({"site": site.site_id, "targets": list(site.targets), "channel": site.channel_id,
                        "probs": [R.kraus_outcome_probability(st, K, site.targets) for K in ch.kraus_ops]})
        key = f"{name}__noiseless"
        arrays[key] = st.amplitudes
        case["kraus_probs"] = {"amps": key, "sites": kop}
        out["cases"][name] = case
        print(name, c.n_qubits, len(c.ops), len(c.sites), file=sys.stderr)

    # throughput_report deterministic columns (m, mode, unique_fraction) on a noiseless demo
    c = build((DEMO / "rychain4.circ").read_text(), (DEMO / "rychain_mixture.noise").read_text())
    spec = R.TrajectorySpec((), 0, None, {"strategy": "bench"})
    rows = R.throughput_report(c, spec, [1, 10, 100, 1000], master_seed=5, naive_prep_cap=8)
    out["throughput_rychain"] = [[r.m, r.mode, r.unique_fraction] for r in rows]

    # CLI run / bench outputs
    cli = {}
    with tempfile.TemporaryDirectory() as tmp:
        tmp = Path(tmp)
        circ, noise = tmp / "c.circ", tmp / "n.noise"
        for cname, ctext, ntext, argv in [
            ("run_probabilistic", (DEMO / "rychain4.circ").read_text(), (DEMO / "rychain_mixture.noise").read_text(),
             ["--strategy", "probabilistic", "--seed", "7", "--nsamples", "100", "--nshots", "1000"]),
            ("run_proportional", W.ghz_repetition(10)[0], W.ghz_repetition(10)[1],
             ["--strategy", "proportional", "--seed", "3", "--nsamples", "300", "--total-shots", "20000"]),
            ("run_cutoff_damped", (DEMO / "teleport5.circ").read_text(), DAMP.format(p=0.2),
             ["--strategy", "cutoff", "--cutoff", "0.01", "--nshots", "50", "--seed", "1"]),
            ("run_probabilistic_damped", (DEMO / "teleport5.circ").read_text(), DAMP.format(p=0.2),
             ["--strategy", "probabilistic", "--nsamples", "80", "--nshots", "50", "--seed", "2"]),
            ("run_band_filtered", W.surface_code_d3(1e-2)[0], W.surface_code_d3(1e-2)[1],
             ["--strategy", "band", "--p-min", "1e-6", "--p-max", "0.5", "--nsamples", "200", "--nshots", "20",
              "--seed", "4", "--filter-qubit", "9", "--filter-qubit", "10", "--filter-gate", "cx"]),
        ]:
            circ.write_text(ctext)
            noise.write_text(ntext)
            d = tmp / cname
            code = ref_cli(["run", "--circuit", str(circ), "--noise", str(noise), "--out", str(d)] + argv)
            cli[cname] = {"circuit": ctext, "noise": ntext, "argv": argv, "code": code}
            if code == 0:
                man = json.loads((d / "manifest.json").read_text())
                cli[cname].update(records=(d / "records.jsonl").read_text(), manifest_core=R.manifest_core(man))
        circ.write_text((DEMO / "ghz4.circ").read_text())
        noise.write_text((DEMO / "depol01.noise").read_text())
        d = tmp / "bench"
        code = ref_cli(["bench", "--circuit", str(circ), "--noise", str(noise), "--seed", "11", "--out", str(d),
                        "--batch-sizes", "1,10,100,1000", "--naive-prep-cap", "4"])
        thr = [line.split(",") for line in (d / "throughput.csv").read_text().splitlines()]
        cli["bench"] = {"circuit": (DEMO / "ghz4.circ").read_text(), "noise": (DEMO / "depol01.noise").read_text(),
                        "code": code, "uniqueness": (d / "uniqueness.csv").read_text(),
                        "throughput_header": thr[0], "throughput_cols": [[r[0], r[1], r[3]] for r in thr[1:]]}
    out["cli"] = cli
    (HERE / "golden_conv.json").write_text(json.dumps(out, indent=1, sort_keys=True))
    np.savez_compressed(HERE / "golden_conv.npz", **arrays)
    print("wrote", HERE / "golden_conv.json", HERE / "golden_conv.npz", file=sys.stderr)


if __name__ == "__main__":
    main()
