"""Native dataset writer (ptsbe_format_records) vs the reference's json.dumps lines.

Host-only: the formatter runs on the CPU side of libptsbe.so, so these run
without a GPU.  The expected text is produced exactly as the reference writes
records.jsonl (ref execute.py:246-259: one json.dumps({"t","b","c"},
separators=(",", ":")) line per record, records of a trajectory sorted by
bitstring, execute.py:181-223; bitstrings format(v, "0{n}b"),
statevector.py:44-53).
"""

import json

import numpy as np
import pytest

from paper_2504_16297_b200.errors import ValidationError
from paper_2504_16297_b200.execute import Dataset, ShotRecord, format_records


def _expected(n, ids, off, idx, cnt):
    lines = []
    for i, t in enumerate(ids):
        lo, hi = off[i], off[i + 1]
        counts = {format(int(v), f"0{n}b"): int(c) for v, c in zip(idx[lo:hi], cnt[lo:hi])}
        for bits in sorted(counts):
            lines.append(json.dumps({"t": int(t), "b": bits, "c": counts[bits]}, separators=(",", ":")) + "\n")
    return "".join(lines).encode()


def _csr(rng, n, n_traj, max_rec, shuffle):
    sizes = np.minimum(rng.integers(0, max_rec + 1, size=n_traj), 1 << min(n, 62))
    off = np.zeros(n_traj + 1, dtype=np.int64)
    np.cumsum(sizes, out=off[1:])
    idx_parts = []
    for s in sizes:
        v = np.sort(rng.choice(1 << n, size=min(int(s), 1 << n), replace=False).astype(np.uint64)) \
            if n <= 20 else np.unique(rng.integers(0, 1 << n, size=int(s), dtype=np.uint64))
        if v.size < s:  # unique() may drop collisions: pad distinct values
            extra = np.setdiff1d(np.arange(s * 2, dtype=np.uint64), v)[: s - v.size]
            v = np.sort(np.concatenate([v, extra]))
        if shuffle:
            rng.shuffle(v)
        idx_parts.append(v)
    idx = np.concatenate(idx_parts) if idx_parts else np.zeros(0, np.uint64)
    cnt = rng.integers(1, 10**7, size=idx.size).astype(np.uint32)
    return off, idx, cnt


@pytest.mark.parametrize("n,shuffle", [(1, False), (5, True), (17, False), (28, True), (64, True)])
def test_matches_reference_lines(n, shuffle):
    rng = np.random.default_rng(n)
    n_traj = 40
    ids = (rng.integers(0, 10**7, size=n_traj) * 100 + np.arange(n_traj)).astype(np.int64) if n % 2 else np.arange(n_traj, dtype=np.int64)
    off, idx, cnt = _csr(rng, n, n_traj, 3 if n == 1 else 50, shuffle)
    got = format_records(n, ids, off, idx, cnt).tobytes()
    assert got == _expected(n, ids, off, idx, cnt)


def test_multithreaded_size_and_order():
    # > 2^16 records takes the threaded path; uneven segments cross the splits
    rng = np.random.default_rng(7)
    n, n_traj = 20, 300
    ids = np.arange(n_traj, dtype=np.int64)
    off, idx, cnt = _csr(rng, n, n_traj, 700, shuffle=True)
    assert off[-1] > 1 << 16
    got = format_records(n, ids, off, idx, cnt).tobytes()
    assert got == _expected(n, ids, off, idx, cnt)


def test_empty_and_zero_length():
    assert format_records(4, [], [0], [], []).size == 0
    assert format_records(4, [3, 4], [0, 0, 0], [], []).size == 0
    got = format_records(3, [0, 1, 2], [0, 0, 2, 2], np.array([5, 1], np.uint64), [2, 7]).tobytes()
    assert got == b'{"t":1,"b":"001","c":7}\n{"t":1,"b":"101","c":2}\n'


def test_invalid_arguments_raise():
    with pytest.raises(ValidationError):
        format_records(0, [0], [0, 1], [0], [1])          # n out of range
    with pytest.raises(ValidationError):
        format_records(3, [0], [0, 1], [8], [1])          # index >= 2^n
    with pytest.raises(ValidationError):
        format_records(3, [0, 1], [0, 2, 1], [1, 2], [1, 1])  # decreasing offsets
    with pytest.raises(ValidationError):
        format_records(3, [-1], [0, 1], [1], [1])         # negative id
    with pytest.raises(ValidationError):
        format_records(3, [0], [0, 5], [1], [1])          # offsets past the arrays


def test_dataset_write_native_equals_json(tmp_path):
    rng = np.random.default_rng(3)
    n, n_traj = 10, 12
    ids = np.arange(n_traj, dtype=np.int64)
    off, idx, cnt = _csr(rng, n, n_traj, 30, shuffle=True)
    recs = []
    for i in range(n_traj):
        counts = {format(int(v), f"0{n}b"): int(c) for v, c in zip(idx[off[i]:off[i + 1]], cnt[off[i]:off[i + 1]])}
        recs.extend(ShotRecord(i, b, counts[b]) for b in sorted(counts))
    plain = Dataset({"n_qubits": n, "trajectories": []}, recs)
    native = Dataset({"n_qubits": n, "trajectories": []}, recs, packed=(n, ids, off, idx, cnt))
    plain.write(tmp_path / "a")
    native.write(tmp_path / "b")
    a = (tmp_path / "a" / "records.jsonl").read_bytes()
    assert a == (tmp_path / "b" / "records.jsonl").read_bytes()
    assert Dataset.read(tmp_path / "b").records == recs


def test_packed_records_sequence_equals_sorted_list():
    from paper_2504_16297_b200.execute import PackedRecords
    rng = np.random.default_rng(11)
    n, n_traj = 12, 25
    ids = np.arange(100, 100 + n_traj, dtype=np.int64)
    off, idx, cnt = _csr(rng, n, n_traj, 40, shuffle=True)
    want = []
    for i in range(n_traj):
        counts = {format(int(v), f"0{n}b"): int(c) for v, c in zip(idx[off[i]:off[i + 1]], cnt[off[i]:off[i + 1]])}
        want.extend(ShotRecord(int(ids[i]), b, counts[b]) for b in sorted(counts))
    pr = PackedRecords(n, ids, off, idx, cnt)
    assert len(pr) == len(want)
    assert list(pr) == want and pr == want
    assert pr[0] == want[0] and pr[-1] == want[-1] and pr[3:9] == want[3:9]
    with pytest.raises(IndexError):
        pr[len(want)]
    assert [r for r in pr if r.trajectory_id == 105] == [r for r in want if r.trajectory_id == 105]
    ds = Dataset({"n_qubits": n, "trajectories": []}, pr, packed=(n, ids, off, idx, cnt))
    assert ds.pooled_counts() == Dataset({}, want).pooled_counts()


def test_packed_validate_matches_record_path():
    from paper_2504_16297_b200.execute import PackedRecords
    rng = np.random.default_rng(5)
    n, n_traj = 9, 6
    ids = np.arange(n_traj, dtype=np.int64)
    off, idx, cnt = _csr(rng, n, n_traj, 20, shuffle=False)
    per = [int(cnt[off[i]:off[i + 1]].sum()) for i in range(n_traj)]
    rows = [{"id": i, "shots": per[i], "status": "ok"} for i in range(n_traj)]
    man = {"n_qubits": n, "trajectories": rows}
    pk = (n, ids, off, idx, cnt)
    Dataset(man, PackedRecords(*pk), packed=pk).validate()
    Dataset(man, list(PackedRecords(*pk))).validate()
    bad = {"n_qubits": n, "trajectories": [dict(r, shots=r["shots"] + (i == 2)) for i, r in enumerate(rows)]}
    for ds in (Dataset(bad, PackedRecords(*pk), packed=pk), Dataset(bad, list(PackedRecords(*pk)))):
        with pytest.raises(ValidationError, match="trajectory 2"):
            ds.validate()
    with pytest.raises(ValidationError):
        Dataset({"n_qubits": n + 1, "trajectories": rows}, PackedRecords(*pk), packed=pk).validate()
    short = {"n_qubits": n, "trajectories": rows[:-1]}
    if off[-1] > off[-2]:
        with pytest.raises(ValidationError, match="unknown trajectory"):
            Dataset(short, PackedRecords(*pk), packed=pk).validate()


def test_packed_pooled_and_per_trajectory_counts():
    from paper_2504_16297_b200.execute import PackedRecords
    rng = np.random.default_rng(21)
    n, n_traj = 6, 30                      # small n: many shared bitstrings across trajectories
    ids = np.arange(n_traj, dtype=np.int64)
    off, idx, cnt = _csr(rng, n, n_traj, 20, shuffle=True)
    pr = PackedRecords(n, ids, off, idx, cnt)
    packed = Dataset({}, pr, packed=(n, ids, off, idx, cnt))
    plain = Dataset({}, list(pr))
    a, b = packed.pooled_counts(), plain.pooled_counts()
    assert a == b and list(a) == list(b)   # same keys in the same order
    for t in (0, 7, 29, 99):
        assert packed.counts_for(t) == plain.counts_for(t)
