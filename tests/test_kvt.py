"""KVT1 reader/writer (paper_2604_08426_b200/kvt.py) against byte streams
written by kvlab's own write_kvt (numerics.py:151-190; tests/golden/tier_io.npz,
made by tests/golden/make_golden.py): identical bytes, identical arrays, and
KvtFormatError exactly where kvlab raises it. CPU only."""

import os

import numpy as np
import pytest

from conftest import golden
from paper_2604_08426_b200 import kvt


@pytest.fixture(scope="module")
def z():
    return golden("tier_io")


@pytest.mark.parametrize("i", [0, 1, 2])
def test_reads_reference_files_and_writes_identical_bytes(z, tmp_path, i):
    blob = z[f"kvt_bytes_{i}"].tobytes()
    ref = z[f"kvt_array_{i}"]
    p = tmp_path / "x.kvt"
    p.write_bytes(blob)
    got = kvt.read_kvt(str(p))
    assert got.dtype == np.float32 and got.shape == ref.shape
    assert np.array_equal(got, ref)
    pinned = kvt.read_kvt(str(p), pinned=True)
    assert tuple(pinned.shape) == ref.shape and np.array_equal(pinned.numpy(), ref)
    q = tmp_path / "y.kvt"
    kvt.write_kvt(str(q), ref)
    assert q.read_bytes() == blob


@pytest.mark.parametrize("name", ["magic", "short_header", "short_extents", "payload", "extra"])
def test_malformed_files_raise_like_reference(z, tmp_path, name):
    assert int(z[f"kvtbad_{name}_raises"]) == 1
    p = tmp_path / "bad.kvt"
    p.write_bytes(z[f"kvtbad_{name}"].tobytes())
    with pytest.raises(kvt.KvtFormatError):
        kvt.read_kvt(str(p))
    assert issubclass(kvt.KvtFormatError, ValueError)


def test_workload_round_trip(tmp_path):
    rng = np.random.default_rng(0)
    wl = kvt.Workload(spec={"n_tokens": 64, "kv_heads": 2}, keys=rng.standard_normal((2, 64, 8), dtype=np.float32),
                      values=rng.standard_normal((2, 64, 8), dtype=np.float32),
                      queries=rng.standard_normal((1, 2, 3, 8), dtype=np.float32),
                      needle_ids=[np.arange(4, dtype=np.int64)])
    d = os.path.join(tmp_path, "wl")
    kvt.save_workload(wl, d)
    back = kvt.load_workload(d)
    assert back.spec == wl.spec
    for f in ("keys", "values", "queries"):
        assert np.array_equal(getattr(back, f), getattr(wl, f))
    assert np.array_equal(back.needle_ids[0], wl.needle_ids[0])
