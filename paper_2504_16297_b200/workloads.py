"""The BASELINE.json configurations as circuit / noise-model TEXT.

Authored in the reference's own text formats (``circuit.py:225-290``,
``circuit.py:373-444``) so the reference parser and this package's parser see
the identical input; SURVEY section 8(d) describes each config.

  1  ghz_repetition(10)      10 q GHZ chain + one ZZ-parity round; h->depolarizing, cx->bit_flip
  2  surface_code_d3()       17 q rotated d=3 syndrome round; depolarizing on every target
  3  random_brickwork(20)    20 q, 10 layers of seeded ry/rz + cx bricks; depolarizing everywhere
  4  steane_blocks(4)        28 q: four [[7,1,3]] blocks, encode + transversal non-Clifford
                             layers + inter-block transversal cx + decode; depolarizing (1q) +
                             bit_flip (cx) on every target
  5  steane_blocks(5)        35 q, same construction (two+ GPUs of sharded state at c64);
     steane_blocks(4, ancillas=6) is its 34-qubit form (CONFIG5_34: fits one B200 sharded
     virtually, 2 x 64 GiB at c64)
"""

from __future__ import annotations

import math

import numpy as np


def _text(n, lines):
    return "\n".join([f"qubits {n}"] + lines) + "\n"


def ghz_repetition(n: int = 10, p1: float = 0.05, p2: float = 0.02):
    """Data qubits 0..d-1 in a GHZ chain, ancillas d..n-1 measure Z_i Z_{i+1}."""
    d = n - (n - 1) // 2 if n > 2 else n
    lines = ["gate h 0"] + [f"gate cx {i} {i + 1}" for i in range(d - 1)]
    for a, anc in enumerate(range(d, n)):
        lines += [f"gate cx {a} {anc}", f"gate cx {a + 1} {anc}"]
    noise = f"rule gate=h qubit=* channel=depolarizing({p1})\nrule gate=cx qubit=* channel=bit_flip({p2})\n"
    return _text(n, lines), noise


def surface_code_d3(p: float = 1e-3):
    """Rotated d=3 surface code: data 0..8 (3x3, row-major), ancillas 9..16."""
    x_stabs = [(0, 1, 3, 4), (4, 5, 7, 8), (2, 5), (3, 6)]
    z_stabs = [(1, 2, 4, 5), (3, 4, 6, 7), (0, 1), (7, 8)]
    xa = list(range(9, 13))
    za = list(range(13, 17))
    lines = [f"gate h {a}" for a in xa]
    for a, stab in zip(xa, x_stabs):
        lines += [f"gate cx {a} {q}" for q in stab]
    for a, stab in zip(za, z_stabs):
        lines += [f"gate cx {q} {a}" for q in stab]
    lines += [f"gate h {a}" for a in xa]
    return _text(17, lines), f"rule gate=* qubit=* channel=depolarizing({p})\n"


def random_brickwork(n: int = 20, layers: int = 10, seed: int = 7, p: float = 1e-3):
    rng = np.random.default_rng(seed)
    lines = []
    for layer in range(layers):
        for q in range(n):
            lines.append(f"gate ry {q} @ {float(rng.uniform(0, 2 * math.pi))!r}")
            lines.append(f"gate rz {q} @ {float(rng.uniform(0, 2 * math.pi))!r}")
        for a in range(layer % 2, n - 1, 2):
            lines.append(f"gate cx {a} {a + 1}")
    return _text(n, lines), f"rule gate=* qubit=* channel=depolarizing({p})\n"


_STEANE_CHECKS = [(0, (2, 4, 6)), (1, (2, 5, 6)), (3, (4, 5, 6))]   # pivot -> targets


def _steane_encode(base: int):
    out = [f"gate h {base + p}" for p, _ in _STEANE_CHECKS]
    for p, ts in _STEANE_CHECKS:
        out += [f"gate cx {base + p} {base + t}" for t in ts]
    return out


def steane_blocks(blocks: int = 4, rounds: int = 7, seed: int = 11, p1: float = 1e-3, p2: float = 1e-3,
                  ancillas: int = 0):
    """``blocks`` [[7,1,3]] blocks (7*blocks qubits): encode, `rounds` x (transversal 1q layer +
    inter-block transversal cx), decode.  >= 300 ops at 4 blocks.  ``ancillas`` extra qubits
    (after the blocks) each extract one Z-type stabilizer of a block (cx from its 4 qubits)
    before the decode -- 4 blocks + 6 ancillas is the 34-qubit size of config 5."""
    n = 7 * blocks + ancillas
    rng = np.random.default_rng(seed)
    lines = []
    for b in range(blocks):
        lines += _steane_encode(7 * b)
    kinds = ("ry", "t", "h", "rz")
    for r in range(rounds):
        kind = kinds[r % len(kinds)]
        for q in range(7 * blocks):
            if kind in ("ry", "rz"):
                lines.append(f"gate {kind} {q} @ {float(rng.uniform(0, 2 * math.pi))!r}")
            else:
                lines.append(f"gate {kind} {q}")
        shift = 1 + r % max(blocks - 1, 1)
        used = set()
        for b in range(blocks):
            partner = (b + shift) % blocks
            if b in used or partner in used or partner == b:
                continue
            used.update((b, partner))
            lines += [f"gate cx {7 * b + i} {7 * partner + i}" for i in range(7)]
    for a in range(ancillas):
        b, (p, ts) = a % blocks, _STEANE_CHECKS[(a // blocks) % 3]
        lines += [f"gate cx {7 * b + q} {7 * blocks + a}" for q in (p,) + ts]
    for b in range(blocks):
        enc = _steane_encode(7 * b)
        lines += list(reversed(enc))     # h and cx are self-inverse
    noise = ("rule gate=cx qubit=* channel=bit_flip({p2})\n"
             "rule gate=* qubit=* channel=depolarizing({p1})\n").format(p1=p1, p2=p2)
    return _text(n, lines), noise


CONFIGS = {
    1: ("ghz_repetition", lambda: ghz_repetition(10)),
    2: ("surface_code_d3", lambda: surface_code_d3()),
    3: ("random_brickwork", lambda: random_brickwork(20)),
    4: ("steane_blocks", lambda: steane_blocks(4)),
    5: ("steane_blocks", lambda: steane_blocks(5)),
    534: ("steane_blocks+ancillas", lambda: steane_blocks(4, ancillas=6)),
}
CONFIG5_34 = 534


def build(config: int, parse_circuit, parse_noise_model, attach_noise):
    """Parse + attach with the given module's functions (ours or the reference's)."""
    _name, make = CONFIGS[config]
    ctext, ntext = make()
    return attach_noise(parse_circuit(ctext), parse_noise_model(ntext))
