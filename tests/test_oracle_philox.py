"""Pins for the RNG contract: published Philox2x32-10
known-answer vectors (Random123 kat_vectors, Salmon et al. SC'11), a library
implementation (libcudacxx cuda::std::philox_engine, i.e. C++26
std::philox_engine, instantiated as Philox2x32-10), the closed form of
`choose`'s buckets, rank64 boundaries, the counter packing, and the two
oracle-side implementations (Python, C++) against each other."""

import glob
import os
import random

import pytest

from oracle import philox as px

# Random123 kat_vectors, "philox2x32 10": ctr0 ctr1 key -> out0 out1
KAT = [
    ((0, 0), 0, (0xFF1DAE59, 0x6CD10DF2)),
    ((0xFFFFFFFF, 0xFFFFFFFF), 0xFFFFFFFF, (0x2C3F628B, 0xAB4FD7AD)),
    ((0x243F6A88, 0x85A308D3), 0x13198A2E, (0xDD7CE038, 0xF62A4C12)),
]


@pytest.mark.parametrize("ctr,key,out", KAT)
def test_philox_kat_python(ctr, key, out):
    assert px.philox2x32_10(ctr, key) == out


@pytest.mark.parametrize("ctr,key,out", KAT)
def test_philox_kat_cpp(oracle_lib, ctr, key, out):
    assert oracle_lib.philox2(ctr, key) == out


def test_philox_python_equals_cpp(oracle_lib):
    rng = random.Random(5)
    for _ in range(2000):
        ctr = tuple(rng.getrandbits(32) for _ in range(2))
        key = rng.getrandbits(32)
        assert px.philox2x32_10(ctr, key) == oracle_lib.philox2(ctr, key)


def test_blocks_python_equals_cpp(oracle_lib):
    """Stream key and step/determinization blocks: Python == C++ oracle."""
    rng = random.Random(6)
    codes = [0x01020004, 0x0305001B, 0x00000000, px.STOP_CODE, px.CRN_WORD]
    for _ in range(500):
        seed, node, s = rng.getrandbits(64), rng.getrandbits(32), rng.getrandbits(32)
        code, t = rng.choice(codes), rng.randrange(64)
        assert px.stream_key(seed, node) == oracle_lib.stream_key(seed, node)
        want = px.det_block(seed, node, code, s) if t == 63 else px.step_block(seed, node, code, s, t)
        assert want == oracle_lib.step_block(seed, node, code, s, t)


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
    """(c0, c1) = (s, t | code12 << 6 | (node mod 2^14) << 18), key = stream_key(seed, node)."""
    seed, node, s = 0xDEADBEEF12345678, 0x12345, 99
    code = 0x02110009                     # target 2, position 17, value key 9
    assert px.code12(code) == (2 << 10) | (17 << 5) | 9
    K = px.philox2x32_10((0x12345678, 0xDEADBEEF), node)[0]
    assert px.stream_key(seed, node) == K
    c1 = 5 | (px.code12(code) << 6) | ((node & 0x3FFF) << 18)
    assert px.step_block(seed, node, code, s, 5) == px.philox2x32_10((s, c1), K)
    c1d = 63 | (px.code12(code) << 6) | ((node & 0x3FFF) << 18)
    assert px.det_block(seed, node, code, s) == px.philox2x32_10((s, c1d), K)
    assert px.code12(px.STOP_CODE) == 0xFFF and px.code12(px.CRN_WORD) == 0xFFE


def test_code12_injective():
    """code12 is injective on every action code of the largest rules (4 seats,
    26-tile lines, keys < 28) plus STOP and the CRN word."""
    seen = {}
    for target in range(4):
        for pos in range(26):
            for v in range(28):
                c = (target << 24) | (pos << 16) | v
                seen.setdefault(px.code12(c), c)
                assert seen[px.code12(c)] == c
    assert px.code12(px.STOP_CODE) not in seen and px.code12(px.CRN_WORD) not in seen
    assert px.code12(px.STOP_CODE) != px.code12(px.CRN_WORD)
    assert max(seen) < (1 << 12)


def test_remainder_is_the_draw_leftover():
    """choose(n, w) * 2^32 + remainder(n, w) == w * n (the joker gap word)."""
    rng = random.Random(9)
    for _ in range(1000):
        n, w = rng.randrange(1, 30), rng.getrandbits(32)
        assert (px.choose(n, w) << 32) + px.remainder(n, w) == w * n


def _cccl_include():
    import site
    for base in site.getsitepackages():
        for p in glob.glob(os.path.join(base, "*", "data", "cccl", "libcudacxx", "include")):
            if os.path.exists(os.path.join(p, "cuda", "std", "__random", "philox_engine.h")):
                return p
    return None


def test_oracle_philox_equals_libcudacxx(oracle_lib, tmp_path):
    """The oracle's Philox2x32-10 equals libcudacxx's cuda::std::philox_engine
    <uint32, 32, 2, 10, 0xD256D193, 0x9E3779B9> (a library implementation,
    compiled host-side) on 20000 random (counter, key) triples."""
    import shutil
    import subprocess
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    inc = _cccl_include()
    if not os.path.exists(nvcc) or inc is None:
        pytest.skip("nvcc or the libcudacxx headers not available")
    exe = str(tmp_path / "cccl_ref")
    src = os.path.join(os.path.dirname(__file__), "native", "cccl_philox2_ref.cu")
    subprocess.check_call([nvcc, "-std=c++17", "-O1", "-I", inc, "-o", exe, src])
    rng = random.Random(77)
    trip = [tuple(rng.getrandbits(32) for _ in range(3)) for _ in range(20000)] + [k[0] + (k[1],) for k in KAT]
    out = subprocess.run([exe], input="\n".join(" ".join(map(str, p)) for p in trip) + "\n",
                         capture_output=True, text=True, check=True).stdout.split("\n")
    for p, line in zip(trip, out):
        ref = tuple(int(x) for x in line.split())
        assert px.philox2x32_10(p[:2], p[2]) == ref
        assert oracle_lib.philox2(p[:2], p[2]) == ref
