"""Pins for oracle Philox4x32-10 and samplers (O6): cuRAND's own Philox round function
(compiled for the host from curand_philox4x32_x.h) and sample moments."""
import os
import shutil
import subprocess

import numpy as np
import pytest

from oracle import sampling

HERE = os.path.dirname(__file__)


@pytest.fixture(scope="module")
def curand_philox(tmp_path_factory):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available")
    exe = str(tmp_path_factory.mktemp("philox") / "philox_host")
    subprocess.check_call([nvcc, "-Wno-deprecated-gpu-targets", "-o", exe,
                           os.path.join(HERE, "tools", "philox_curand_host.cu")])
    return exe


def test_philox_matches_curand(curand_philox):
    rng = np.random.default_rng(11)
    for seed in (0, 1, 2, 0xDEADBEEFCAFEF00D, 2 ** 64 - 1):
        key = (seed & 0xFFFFFFFF, seed >> 32)
        ctrs = [(0, 0, 0, 0), (1, 2, 3, 4), (16383, 783, 5, 8)] + \
               [tuple(int(v) for v in rng.integers(0, 2 ** 32, 4, dtype=np.uint64)) for _ in range(40)]
        inp = "".join(f"{a} {b} {c} {d}\n" for a, b, c, d in ctrs)
        out = subprocess.run([curand_philox, str(key[0]), str(key[1])], input=inp, capture_output=True,
                             text=True, check=True).stdout.split("\n")
        for ctr, line in zip(ctrs, out):
            want = [int(v) for v in line.split()]
            got = [int(v) for v in sampling.philox4x32_10(ctr, key)]
            assert got == want, (seed, ctr)


def test_philox_known_zero_vector():
    # Random123 known-answer for philox4x32-10 with ctr=0, key=0 (also what cuRAND returns).
    assert [hex(int(v)) for v in sampling.philox4x32_10([0, 0, 0, 0], [0, 0])] == \
        ["0x6627e8d5", "0xe169c58d", "0xbc57ac4c", "0x9b00dbd8"]


def test_uniform_sampler_definition():
    q = 0xFFFFFFFFFFE8001
    got = sampling.uniform(64, 5, 3, 2, sampling.TAG_RLK_A, q)
    for k in range(64):
        x = [int(v) for v in sampling.philox4x32_10([k, 3, 2, sampling.TAG_RLK_A], [5, 0])]
        u = x[0] | (x[1] << 32) | (x[2] << 64) | (x[3] << 96)
        assert int(got[k]) == u % q


def test_ternary_and_cbd_moments():
    n = 1 << 16
    t = sampling.ternary(n, 1, 0, sampling.TAG_S)
    assert set(np.unique(t).tolist()) == {-1, 0, 1}
    for v in (-1, 0, 1):
        assert abs(np.mean(t == v) - 1 / 3) < 0.01
    e = sampling.cbd(n, 1, 0, sampling.TAG_PK_E)
    assert np.abs(e).max() <= 21
    assert abs(e.mean()) < 0.05
    assert abs(e.var() - 10.5) / 10.5 < 0.02


def test_cbd_definition():
    e = sampling.cbd(32, 9, 4, sampling.TAG_ENC_E0)
    for k in range(32):
        x = [int(v) for v in sampling.philox4x32_10([k, 4, 0, sampling.TAG_ENC_E0], [9, 0])]
        assert e[k] == bin(x[0] & 0x1FFFFF).count("1") - bin(x[1] & 0x1FFFFF).count("1")
    t = sampling.ternary(32, 9, 4, sampling.TAG_ENC_V)
    for k in range(32):
        x = [int(v) for v in sampling.philox4x32_10([k, 4, 0, sampling.TAG_ENC_V], [9, 0])]
        assert t[k] == x[0] % 3 - 1
