"""CPU-side checks of the C-ABI boundary (no GPU needed): the library loads,
exports every symbol include/kvb.h declares, maps reference ValueError
conditions to KVB_EINVAL, and its host-side outlier chooser equals the
reference's greedy fill (kvstore.py:181-190)."""

import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "kvb.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2604_08426_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):
        from paper_2604_08426_b200 import build

        build.build()
    return _lib.load()


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(kvb_[a-z0-9_]+)\s*\(", text)))


def test_exports_every_declared_symbol(lib):
    names = header_functions()
    assert len(names) >= 25
    for name in names:
        assert hasattr(lib, name), f"libkvb.so does not export {name}"


def test_binding_covers_header():
    from paper_2604_08426_b200 import _lib

    bound = {n for n, _, _ in _lib.SIGNATURES}
    assert set(header_functions()) == bound


def test_abi_version(lib):
    assert lib.kvb_abi_version() == 1


def test_invalid_store_is_einval(lib):
    from paper_2604_08426_b200 import _lib

    d = _lib.StoreDesc()
    d.batch, d.n_tokens, d.kv_heads, d.head_dim, d.chunk_size = 1, 0, 1, 4, 1
    d.max_resident = 1
    h = C.c_void_p()
    st = lib.kvb_store_create(C.byref(d), C.byref(h))
    assert st == _lib.KVB_EINVAL
    assert b"at least one token" in lib.kvb_last_error()
    d.n_tokens, d.chunk_size = 8, 0
    assert lib.kvb_store_create(C.byref(d), C.byref(h)) == _lib.KVB_EINVAL
    with pytest.raises(ValueError):
        _lib.check(_lib.KVB_EINVAL, "x")


@pytest.mark.parametrize("seed", range(20))
def test_choose_outliers_matches_reference_greedy(lib, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 400))
    cs = int(rng.integers(1, 12))
    C_ = -(-n // cs)
    budget = int(rng.integers(0, 64))
    per = rng.standard_normal(C_)
    if seed % 3 == 0:  # ties exercise the stable order
        per = np.round(per, 1)
    out = np.zeros(C_, np.int32)
    cnt = C.c_int32()
    assert lib.kvb_choose_outliers(per.ctypes.data_as(C.c_void_p), C_, n, cs, budget,
                                   out.ctypes.data_as(C.c_void_p), C.byref(cnt)) == 0
    got = tuple(out[: cnt.value].tolist())
    # kvstore.py:181-190 restated
    order = [0] + [int(c) for c in np.argsort(per, kind="stable") if c != 0]
    chosen, used = [], 0
    if budget > 0:
        for c in order:
            size = min(cs, n - c * cs)
            if used + size <= budget:
                chosen.append(c)
                used += size
    assert got == tuple(sorted(chosen))


def test_codebooks_shipped_match_reference():
    from conftest import golden
    from paper_2604_08426_b200 import schemes

    z = golden("codecs")
    for bits in (1, 2, 4):
        assert np.array_equal(schemes.higgs_codebook(2, 2 ** (2 * bits), 0), z[f"codebook_b{bits}"])
    assert np.array_equal(schemes.hadamard_signs(1024, 0), z["signs_1024_s0"])


def test_scheme_strings_round_trip():
    from paper_2604_08426_b200 import schemes as S

    for t in ("none", "higgs2", "higgs:d=2,n=256,group=256,seed=3", "svd:rank=160,dim=1024"):
        s = S.scheme_from_string(t)
        assert S.scheme_from_string(S.scheme_to_string(s)) == s
    assert S.bits_per_key(S.scheme_none(), 8) == 2
    assert S.bits_per_key(S.scheme_higgs(4), 2) == 2
    assert S.bits_per_key(S.scheme_higgs(2), 1) == 2
    assert S.bits_per_key(S.scheme_higgs(4), 8, S.scheme_higgs(1)) == S.Fraction(3, 2)
