"""ORACLE -- test infrastructure only.

Plain, slow, obviously-correct CPU implementations of what the batched Da Vinci
Code rollout computes:

  * oracle/philox.py  -- Philox2x32-10, stream key, counter layout, choose,
                         rank64 (the RNG contract);
  * oracle/game.py    -- list-based rules, canonical determinization
                         (count + unrank) and the Philox-driven playout (Python);
  * oracle/exact.py   -- exact rational win probabilities (tiny tile sets);
  * oracle/oracle.cpp -- the same playout in scalar single-threaded C++17
                         (fast enough for full-size parity and the CPU baseline);
  * oracle/fixtures.py -- the seeded position generator (deals, random play)
                         that writes the committed fixtures/*.json.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline /
`--impl reference` legs may import this package.  The product path
(`paper_2403_10720_b200/`) never imports it, and the two share no code.

Parity status: every function here is pinned by a `-m "not gpu"` test
(tests/test_oracle_*.py) -- Random123 KATs, brute-force enumeration,
hand-worked endgames from tests/golden/, exact probabilities, invariants.
"""

import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force=False):
    """Compile oracle.cpp -> liboracle.so (g++ -O2, scalar, no intrinsics)."""
    src = os.path.join(_HERE, "oracle.cpp")
    if not force and os.path.exists(_SO) and os.path.getmtime(_SO) >= os.path.getmtime(src):
        return _SO
    tmp = _SO + ".tmp.%d" % os.getpid()
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o", tmp, src])
    os.replace(tmp, _SO)
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P, U32, U64, I32 = ctypes.POINTER, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int32
        L.oracle_last_error.restype = ctypes.c_char_p
        L.oracle_philox2.argtypes = [P(U32), U32, P(U32)]
        L.oracle_stream_key.argtypes = [U64, U32]
        L.oracle_stream_key.restype = U32
        L.oracle_step_block.argtypes = [U64, U32, U32, U32, U32, P(U32)]
        L.oracle_count.argtypes = [P(I32), P(U64)]
        L.oracle_unrank.argtypes = [P(I32), U64, P(I32), I32, P(I32)]
        L.oracle_legal.argtypes = [P(I32), P(U32), I32, P(I32)]
        L.oracle_rollout.argtypes = [P(I32), P(U32), I32, U64, U32, U64, U64, P(U64)]
        L.oracle_rollout_flags.argtypes = [P(I32), P(U32), I32, U64, U32, U64, U64, P(U64), I32]
        L.oracle_playout.argtypes = [P(I32), U32, U64, U32, U32, P(I32)]
        L.oracle_rollout_fixed.argtypes = [P(I32), P(U32), P(U64), I32, U64, U32, U64, U64, P(U64)]
        L.oracle_rollout_path.argtypes = [P(I32), P(U32), I32, P(U32), I32, U64, U32, U64, U64, P(U64), P(U64)]
        _lib = L
    return _lib


def flatten(obs_json):
    """Fixture JSON -> the oracle's flat int32 observation (see oracle.cpp)."""
    r = obs_json["rules"]
    R = int(r.get("ranks", 12))
    out = [int(r["players"]), R, int(r.get("jokers", 0)), int(r.get("consecutive", 1)),
           int(obs_json["viewer"]), int(obs_json["pool_size"]),
           int(obs_json.get("pending", -1)), int(obs_json.get("correct_this_turn", 0))]
    for line in obs_json["lines"]:
        out.append(len(line))
        for t in line:
            c = 0 if t["color"] == "B" else 1
            v = t.get("value")
            key = -1 if v is None else (2 * R + c if v == "J" else 2 * int(v) + c)
            out += [c, key, 1 if t.get("revealed", False) else 0]
    return (ctypes.c_int32 * len(out))(*out)


def _check(rc):
    if rc < 0:
        raise RuntimeError("oracle error %d: %s" % (rc, lib().oracle_last_error().decode()))
    return rc


def philox2(ctr, key):
    """Philox2x32-10 of the C++ oracle: ctr 2 x u32, key u32 -> 2 x u32."""
    c = (ctypes.c_uint32 * 2)(*ctr)
    o = (ctypes.c_uint32 * 2)()
    lib().oracle_philox2(c, key, o)
    return tuple(o)


def stream_key(seed, node_id):
    return lib().oracle_stream_key(seed, node_id)


def step_block(seed, node_id, code, s, t):
    """B_t (t = 63: the determinization block D) of the C++ oracle."""
    o = (ctypes.c_uint32 * 2)()
    lib().oracle_step_block(seed, node_id, code, s, t, o)
    return tuple(o)


def count(obs_json):
    n = ctypes.c_uint64()
    _check(lib().oracle_count(flatten(obs_json), ctypes.byref(n)))
    return n.value


def unrank(obs_json, rho):
    buf = (ctypes.c_int32 * 128)()
    n = ctypes.c_int32()
    _check(lib().oracle_unrank(flatten(obs_json), rho, buf, 128, ctypes.byref(n)))
    return list(buf[:n.value])


def legal(obs_json):
    buf = (ctypes.c_uint32 * 4096)()
    n = ctypes.c_int32()
    _check(lib().oracle_legal(flatten(obs_json), buf, 4096, ctypes.byref(n)))
    return list(buf[:n.value])


def rollout(obs_json, codes, seed, node_id, s0, s1, crn=False, informed=False):
    """hist[a][w] (list of lists) for sims [s0, s1); crn = common
    determinizations across actions; informed = order-aware
    playout policy (§R10)."""
    P = int(obs_json["rules"]["players"])
    A = len(codes)
    c = (ctypes.c_uint32 * max(A, 1))(*codes)
    h = (ctypes.c_uint64 * max(A * P, 1))()
    flags = (1 if crn else 0) | (2 if informed else 0)
    _check(lib().oracle_rollout_flags(flatten(obs_json), c, A, seed, node_id, s0, s1, h, flags))
    return [list(h[a * P:(a + 1) * P]) for a in range(A)]


def rollout_fixed(obs_json, codes, rhos, seed, node_id, s0, s1):
    """The md ablation batch: hist[i][w] for child i =
    (determinization rhos[i], action codes[i]), sims [s0, s1)."""
    P = int(obs_json["rules"]["players"])
    A = len(codes)
    c = (ctypes.c_uint32 * max(A, 1))(*codes)
    r = (ctypes.c_uint64 * max(A, 1))(*rhos)
    h = (ctypes.c_uint64 * max(A * P, 1))()
    _check(lib().oracle_rollout_fixed(flatten(obs_json), c, r, A, seed, node_id, s0, s1, h))
    return [list(h[a * P:(a + 1) * P]) for a in range(A)]


def playout(obs_json, code, seed, node_id, s):
    """(winner, #decisions) of one playout."""
    st = ctypes.c_int32()
    w = _check(lib().oracle_playout(flatten(obs_json), code, seed, node_id, s, ctypes.byref(st)))
    return w, st.value


def rollout_path(obs_json, path, codes, seed, node_id, s0, s1):
    """Deep-tree batch: (hist[a][w], voids[a]) for forced path + codes[a]."""
    if not path:
        return rollout(obs_json, codes, seed, node_id, s0, s1), [0] * len(codes)
    P = int(obs_json["rules"]["players"])
    A = len(codes)
    c = (ctypes.c_uint32 * max(A, 1))(*codes)
    p = (ctypes.c_uint32 * len(path))(*path)
    h = (ctypes.c_uint64 * max(A * P, 1))()
    v = (ctypes.c_uint64 * max(A, 1))()
    _check(lib().oracle_rollout_path(flatten(obs_json), p, len(path), c, A, seed, node_id, s0, s1, h, v))
    return [list(h[a * P:(a + 1) * P]) for a in range(A)], list(v[:A])
