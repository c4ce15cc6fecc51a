"""TTB1 core files, host only.  The fixture bytes are assembled
here field by field from the SPEC text, independently of ttb1.save."""
import struct

import numpy as np
import pytest

from paper_1511_06029_b200 import ttb1


def _handmade(tmp_path):
    # d = 2 operator, ranks [1, 2, 1]; core 1 value = 100*a + 10*(2i+j) + b
    g1 = np.array([[[[1.0 * (10 * (2 * i + j) + b) for b in range(2)] for j in range(2)] for i in range(2)]])
    g2 = np.array([[[[100.0 * a + 10 * (2 * i + j)] for j in range(2)] for i in range(2)] for a in range(2)])
    raw = b"TTB1" + struct.pack("<II", 2, 1) + struct.pack("<2I", 2, 2) + struct.pack("<2I", 2, 2) \
        + struct.pack("<3I", 1, 2, 1)
    raw += struct.pack("<8d", *[10 * p + b for p in range(4) for b in range(2)])
    raw += struct.pack("<8d", *[100 * a + 10 * p for a in range(2) for p in range(4)])
    path = tmp_path / "op.ttb1"
    path.write_bytes(raw)
    return path, [g1, g2]


def test_load_handmade_operator(tmp_path):
    path, ref = _handmade(tmp_path)
    ranks, cores = ttb1.load_operator(path)
    assert ranks == [1, 2, 1]
    for c, r in zip(cores, ref):
        np.testing.assert_array_equal(c, r)
    # (i, j) flattened row-digit major: core 1 entry [0, i=1, j=0, b=1] = 10*2 + 1
    assert cores[0][0, 1, 0, 1] == 21.0


def test_round_trip_and_vectors(tmp_path):
    rng = np.random.default_rng(0)
    ranks = [1, 3, 4, 2, 1]
    cores = [rng.standard_normal((ranks[k], 2, 2, ranks[k + 1])) for k in range(4)]
    ttb1.save(tmp_path / "a.ttb1", cores)
    r2, c2 = ttb1.load_operator(tmp_path / "a.ttb1")
    assert r2 == ranks
    for a, b in zip(cores, c2):
        np.testing.assert_array_equal(a, b)
    vec = [rng.standard_normal((ranks[k], 2, ranks[k + 1])) for k in range(4)]
    ttb1.save(tmp_path / "v.ttb1", vec, vector=True)
    kind, rv, cv = ttb1.load(tmp_path / "v.ttb1")
    assert kind == "vector" and rv == ranks
    with pytest.raises(ValueError):
        ttb1.load_operator(tmp_path / "v.ttb1")


def test_rejects_mismatched_files(tmp_path):
    path, _ = _handmade(tmp_path)
    raw = path.read_bytes()
    for bad in (raw[:-8], raw + b"\0" * 8, b"TTB2" + raw[4:], raw[:10]):
        p = tmp_path / "bad.ttb1"
        p.write_bytes(bad)
        with pytest.raises(ValueError):
            ttb1.load(p)
    # non-binary modes load but are refused as a QTT operator for this library
    rng = np.random.default_rng(1)
    ttb1.save(tmp_path / "m3.ttb1", [rng.standard_normal((1, 3, 3, 1))])
    ttb1.load(tmp_path / "m3.ttb1")
    with pytest.raises(ValueError):
        ttb1.load_operator(tmp_path / "m3.ttb1")
