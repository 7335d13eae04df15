"""The C-ABI library loads and exports every symbol include/edl.h declares (no GPU
compute), and its host-side parameter derivation agrees with the oracle's."""
import ctypes
import os
import re

import pytest

from oracle.params import params_from_depth as oracle_params

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "edl.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(edl_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2110_13638_b200 import build
    build.build()
    return ctypes.CDLL(build.LIB)


def test_every_declared_symbol_exported(lib):
    names = _declared()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n


def test_binding_covers_header():
    from paper_2110_13638_b200 import edl
    assert set(_declared()) == set(edl.EXPORTED)


@pytest.mark.parametrize("depth", [0, 1, 2, 3, 4, 5])
def test_params_match_oracle(depth):
    from paper_2110_13638_b200 import edl
    p = edl.params_from_depth(depth)
    o = oracle_params(depth)
    assert p.n == o.n and p.chain_bits == o.bits
    assert p.qs == o.q and int(p.p_special) == o.p_special and p.psis == o.psi


def test_microbench_chains_match_oracle():
    from paper_2110_13638_b200 import edl
    from oracle.params import make_params, microbench_bits
    for logn in (13, 14):
        for nd in (3, 6, 12):
            bits = microbench_bits(nd)
            p = edl.params_from_bits(logn, bits)
            o = make_params(1 << logn, bits)
            assert p.qs == o.q and p.psis == o.psi


def test_bad_params_rejected():
    from paper_2110_13638_b200 import edl
    with pytest.raises(edl.ArgError):
        edl.params_from_depth(-1)
    assert edl.cts_bytes(3, 2, 13) == 3 * 2 * 3 * 8192 * 8
