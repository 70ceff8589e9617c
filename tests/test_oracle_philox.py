"""Pins for the RNG contract: published Philox4x32-10
known-answer vectors (Random123 kat_vectors, Salmon et al. SC'11), the closed
form of `choose`'s buckets, rank64 boundaries, and the two oracle-side
implementations (Python, C++) against each other."""

import os
import random

import pytest

from oracle import philox as px

KAT = [
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


@pytest.mark.parametrize("ctr,key,out", KAT)
def test_philox_kat_python(ctr, key, out):
    assert px.philox4x32_10(ctr, key) == out


@pytest.mark.parametrize("ctr,key,out", KAT)
def test_philox_kat_cpp(oracle_lib, ctr, key, out):
    assert oracle_lib.philox_block(ctr, key) == out


def test_philox_python_equals_cpp(oracle_lib):
    rng = random.Random(5)
    for _ in range(2000):
        ctr = tuple(rng.getrandbits(32) for _ in range(4))
        key = tuple(rng.getrandbits(32) for _ in range(2))
        assert px.philox4x32_10(ctr, key) == oracle_lib.philox_block(ctr, key)


def test_seed_key_split():
    assert px.seed_key(0x0123456789ABCDEF) == (0x89ABCDEF, 0x01234567)


@pytest.mark.parametrize("n", [1, 2, 3, 5, 7, 22, 104, 1000003, (1 << 32) - 1])
def test_choose_buckets_closed_form(n):
    """Bucket i = {w : floor(w n / 2^32) = i} = [ceil(i 2^32/n), ceil((i+1) 2^32/n)),
    so every bucket holds floor(2^32/n) or ceil(2^32/n) words."""
    M = 1 << 32
    assert px.choose(n, 0) == 0
    assert px.choose(n, M - 1) == n - 1
    idx = range(n) if n <= 1000 else [0, 1, 2, n // 2, n - 2, n - 1]
    for i in idx:
        lo = -(-i * M // n)
        hi = -(-(i + 1) * M // n)
        assert hi - lo in (M // n, -(-M // n))
        assert px.choose(n, lo) == i
        assert px.choose(n, hi - 1) == i
        if lo > 0:
            assert px.choose(n, lo - 1) == i - 1


@pytest.mark.parametrize("N", [1, 2, 3, 262, 760000, (1 << 45) - 1, (1 << 64) - 1])
def test_rank64_boundaries(N):
    M = 0xFFFFFFFF
    assert px.rank64(N, 0, 0) == 0
    assert px.rank64(N, M, M) == N - 1
    # monotone in the 64-bit word, hits rho exactly at ceil(rho 2^64 / N)
    for rho in (0, N // 3, N - 1):
        x = -(-rho * (1 << 64) // N)
        assert px.rank64(N, x & M, x >> 32) == rho
        if x > 0:
            x -= 1
            assert px.rank64(N, x & M, x >> 32) == rho - 1


def test_counter_layout():
    """D uses ctr.x = 0xFFFFFFFF, step t uses ctr.x = t; (y, z, w) = (s, code, node)."""
    seed, node, code, s = 0xDEADBEEF12345678, 7, 0x01020304, 99
    key = px.seed_key(seed)
    assert px.det_block(seed, node, code, s) == px.philox4x32_10((0xFFFFFFFF, s, code, node), key)
    assert px.step_block(seed, node, code, s, 5) == px.philox4x32_10((5, s, code, node), key)


def test_oracle_philox_equals_curand(oracle_lib, tmp_path):
    """The oracle's Philox4x32-10 equals cuRAND's curand_Philox4x32_10 (a
    library implementation, compiled host-side from the CUDA toolkit header)
    on 20000 random (counter, key) pairs."""
    import shutil
    import subprocess
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc) and not shutil.which("nvcc"):
        pytest.skip("nvcc not available")
    exe = str(tmp_path / "curand_ref")
    src = os.path.join(os.path.dirname(__file__), "native", "curand_philox_ref.cu")
    subprocess.check_call([nvcc, "-O1", "-o", exe, src])
    rng = random.Random(77)
    pairs = [tuple(rng.getrandbits(32) for _ in range(6)) for _ in range(20000)]
    out = subprocess.run([exe], input="\n".join(" ".join(map(str, p)) for p in pairs) + "\n",
                         capture_output=True, text=True, check=True).stdout.split("\n")
    for p, line in zip(pairs, out):
        ref = tuple(int(x) for x in line.split())
        assert px.philox4x32_10(p[:4], p[4:]) == ref
        assert oracle_lib.philox_block(p[:4], p[4:]) == ref
