"""Thin ctypes binding of libdvc.so (include/dvc.h) -- argument marshalling only.

Every step of the hot path runs in the CUDA kernels behind the C-ABI; there is
no Python or CPU fallback: if libdvc.so is missing, `lib()` raises, and if no
CUDA device is usable the rollout calls raise DvcError(DVC_E_CUDA).
PyTorch is used only for device memory and streams (the *_async forms take
torch CUDA tensors).
"""

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# DVC_DEBUG=1 selects the debug build (device-side invariant checks);
# DVC_LIB=<file name in this directory> selects another build (A/B timing)
LIB_PATH = os.path.join(HERE, os.environ.get("DVC_LIB") or
                        ("libdvc_debug.so" if os.environ.get("DVC_DEBUG") == "1" else "libdvc.so"))

DVC_OK = 0
ERRORS = {-1: "DVC_E_CONFIG", -2: "DVC_E_PROTOCOL", -3: "DVC_E_ILLEGAL",
          -4: "DVC_E_INCONSISTENT", -5: "DVC_E_CAPACITY", -6: "DVC_E_CUDA"}
STOP = 0xFFFFFFFF
JOKER = 0xFE
HIDDEN = 0xFF

# every symbol include/dvc.h declares
EXPORTS = ["dvc_state_encode", "dvc_state_query", "dvc_legal_actions", "dvc_rollout_batch",
           "dvc_rollout_batch_ex", "dvc_rollout_path_ex", "dvc_rollout_batch_async", "dvc_rollout_trace_async",
           "dvc_rollout_batch_flags_ex", "dvc_rollout_batch_flags_async", "dvc_rollout_batch_fixed_ex",
           "dvc_sample_determinizations", "dvc_mcts_search", "dvc_mcts_search_cb", "dvc_md_search",
           "dvc_set_option", "dvc_get_option", "dvc_debug_counters", "dvc_launch_count", "dvc_transfer_bytes",
           "dvc_last_error",
           "dvc_shutdown"]


class DvcError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__("%s (%d): %s" % (ERRORS.get(code, "?"), code, msg))
        self.code = code


class _Rules(ctypes.Structure):
    _fields_ = [("players", ctypes.c_int32), ("ranks", ctypes.c_int32),
                ("jokers", ctypes.c_int32), ("consecutive", ctypes.c_int32)]


class _TileObs(ctypes.Structure):
    _fields_ = [("color", ctypes.c_uint8), ("value", ctypes.c_uint8),
                ("revealed", ctypes.c_uint8), ("_pad", ctypes.c_uint8)]


class _Observation(ctypes.Structure):
    _fields_ = [("rules", _Rules), ("viewer", ctypes.c_int32), ("line_len", ctypes.c_int32 * 4),
                ("line", (_TileObs * 26) * 4), ("pool_size", ctypes.c_int32),
                ("pending", ctypes.c_int32), ("correct_this_turn", ctypes.c_int32)]


class _State(ctypes.Structure):
    _fields_ = [("opaque", ctypes.c_uint64 * 128)]


class _SearchParams(ctypes.Structure):
    _fields_ = [("c", ctypes.c_double), ("max_depth", ctypes.c_int32), ("expansions", ctypes.c_int32),
                ("sims_per_child", ctypes.c_uint64), ("seed", ctypes.c_uint64), ("flat", ctypes.c_int32),
                ("device", ctypes.c_int32), ("flags", ctypes.c_uint32), ("_pad", ctypes.c_uint32)]


class _MdParams(ctypes.Structure):
    _fields_ = [("c", ctypes.c_double), ("n_det", ctypes.c_int32), ("expansions", ctypes.c_int32),
                ("sims_per_child", ctypes.c_uint64), ("seed", ctypes.c_uint64), ("device", ctypes.c_int32),
                ("_pad", ctypes.c_uint32)]


class _ActionStat(ctypes.Structure):
    _fields_ = [("code", ctypes.c_uint32), ("_pad", ctypes.c_uint32), ("visits", ctypes.c_uint64),
                ("wins", ctypes.c_uint64)]


class _StateInfo(ctypes.Structure):
    _fields_ = [("players", ctypes.c_int32), ("ranks", ctypes.c_int32), ("jokers", ctypes.c_int32),
                ("consecutive", ctypes.c_int32), ("viewer", ctypes.c_int32),
                ("pool_size", ctypes.c_int32), ("n_legal", ctypes.c_int32), ("_pad", ctypes.c_int32),
                ("n_det", ctypes.c_uint64)]


# dvc_batch_fn (include/dvc.h): (ctx, path, path_len, actions, n_actions, seed,
# node_id, sim_begin, sim_end, flags, hist, voids) -> status
BATCH_FN = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint32), ctypes.c_int32,
                            ctypes.POINTER(ctypes.c_uint32), ctypes.c_int32, ctypes.c_uint64, ctypes.c_uint32,
                            ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint64),
                            ctypes.POINTER(ctypes.c_uint64))

_lib = None


def lib():
    """Load libdvc.so (built in-tree by __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError("libdvc.so not built: run `python -m paper_2403_10720_b200.build` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        P, U8, U32, U64, I32, I64 = (ctypes.POINTER, ctypes.c_uint8, ctypes.c_uint32, ctypes.c_uint64,
                                     ctypes.c_int32, ctypes.c_int64)
        VP = ctypes.c_void_p
        L.dvc_state_encode.argtypes = [P(_Observation), P(_State)]
        L.dvc_state_query.argtypes = [P(_State), P(_StateInfo)]
        L.dvc_legal_actions.argtypes = [P(_State), P(U32), I32, P(I32)]
        L.dvc_rollout_batch.argtypes = [P(_State), P(U32), I32, U64, U64, P(U64)]
        L.dvc_rollout_batch_ex.argtypes = [P(_State), P(U32), I32, U64, U32, U64, U64, P(U64), P(U64), I32]
        L.dvc_rollout_path_ex.argtypes = [P(_State), P(U32), I32, P(U32), I32, U64, U32, U64, U64, P(U64), P(U64),
                                          I32]
        L.dvc_rollout_batch_async.argtypes = [P(_State), P(U32), I32, U64, U32, U64, U64, VP, VP, I32, VP]
        L.dvc_rollout_trace_async.argtypes = [P(_State), P(U32), I32, U64, U32, U64, U64, VP, VP, I32, VP]
        L.dvc_rollout_batch_flags_ex.argtypes = [P(_State), P(U32), I32, U64, U32, U64, U64, U32, P(U64), I32]
        L.dvc_rollout_batch_fixed_ex.argtypes = [P(_State), P(U32), P(U64), I32, U64, U32, U64, U64, P(U64), I32]
        L.dvc_rollout_batch_flags_async.argtypes = [P(_State), P(U32), I32, U64, U32, U64, U64, U32, VP, I32, VP]
        L.dvc_mcts_search.argtypes = [P(_State), P(_SearchParams), P(_ActionStat), I32, P(I32), P(U32)]
        L.dvc_mcts_search_cb.argtypes = [P(_State), P(_SearchParams), BATCH_FN, VP, P(_ActionStat), I32, P(I32),
                                         P(U32)]
        L.dvc_md_search.argtypes = [P(_State), P(_MdParams), P(_ActionStat), I32, P(I32), P(U32), P(I32)]
        L.dvc_sample_determinizations.argtypes = [P(_State), U64, U32, U32, I32, P(U64)]
        L.dvc_debug_counters.argtypes = [I32, P(U32)]
        L.dvc_set_option.argtypes = [ctypes.c_char_p, I64]
        L.dvc_get_option.argtypes = [ctypes.c_char_p, P(I64)]
        L.dvc_launch_count.argtypes = [I32]
        L.dvc_transfer_bytes.argtypes = [I32, P(U64), P(U64)]
        L.dvc_launch_count.restype = U64
        L.dvc_last_error.restype = ctypes.c_char_p
        L.dvc_shutdown.restype = None
        for name in EXPORTS:
            if name not in ("dvc_launch_count", "dvc_last_error", "dvc_shutdown"):
                getattr(L, name).restype = I32
        _lib = L
    return _lib


def _check(rc):
    if rc != DVC_OK:
        raise DvcError(rc, lib().dvc_last_error().decode())


def observation(obs_json):
    """Fixture JSON (SPEC:191 tile shape + pending/correct_this_turn) -> dvc_observation."""
    o = _Observation()
    r = obs_json["rules"]
    o.rules.players = int(r["players"])
    o.rules.ranks = int(r.get("ranks", 12))
    o.rules.jokers = int(r.get("jokers", 0))
    o.rules.consecutive = int(r.get("consecutive", 1))
    o.viewer = int(obs_json["viewer"])
    lines = obs_json["lines"]
    if len(lines) > 4:
        raise ValueError("at most 4 players")
    for p, line in enumerate(lines):
        if len(line) > 26:
            raise ValueError("line too long")
        o.line_len[p] = len(line)
        for i, t in enumerate(line):
            e = o.line[p][i]
            e.color = 0 if t["color"] == "B" else 1
            v = t.get("value")
            e.value = HIDDEN if v is None else (JOKER if v == "J" else int(v))
            e.revealed = 1 if t.get("revealed", False) else 0
    o.pool_size = int(obs_json["pool_size"])
    o.pending = int(obs_json.get("pending", -1))
    o.correct_this_turn = int(obs_json.get("correct_this_turn", 0))
    return o


class State:
    """An encoded root (dvc_state): immutable, pointer-free, picklable bytes."""

    def __init__(self, raw):
        self._s = raw

    @staticmethod
    def encode(obs_json):
        s = _State()
        _check(lib().dvc_state_encode(ctypes.byref(observation(obs_json)), ctypes.byref(s)))
        return State(s)

    def to_bytes(self):
        return bytes(self._s)

    @staticmethod
    def from_bytes(b):
        return State(_State.from_buffer_copy(b))

    @property
    def info(self):
        i = _StateInfo()
        _check(lib().dvc_state_query(ctypes.byref(self._s), ctypes.byref(i)))
        return {k: getattr(i, k) for k, _ in _StateInfo._fields_ if not k.startswith("_")}

    @property
    def players(self):
        return self.info["players"]

    def legal_actions(self):
        n = ctypes.c_int32()
        _check(lib().dvc_legal_actions(ctypes.byref(self._s), None, 0, ctypes.byref(n)))
        buf = (ctypes.c_uint32 * max(n.value, 1))()
        _check(lib().dvc_legal_actions(ctypes.byref(self._s), buf, n.value, ctypes.byref(n)))
        return list(buf[:n.value])


def encode(obs_json):
    return State.encode(obs_json)


def _codes(actions):
    a = np.ascontiguousarray(np.asarray(actions, dtype=np.uint32))
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))


def rollout_batch(state, actions, n_sims, seed):
    """wins[a] of the viewer over sims [0, n_sims), node 0 (blocking, host output)."""
    a, ap = _codes(actions)
    wins = np.zeros(len(a), dtype=np.uint64)
    _check(lib().dvc_rollout_batch(ctypes.byref(state._s), ap, len(a), n_sims, seed,
                                   wins.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))))
    return wins


FLAG_CRN, FLAG_INFORMED = 1, 2


def _flags(crn, informed):
    return (FLAG_CRN if crn else 0) | (FLAG_INFORMED if informed else 0)


def rollout_batch_ex(state, actions, seed, node_id, sim_begin, sim_end, device=-1, crn=False, informed=False):
    """hist[a, w] (numpy uint64, host) for sims [sim_begin, sim_end) (blocking).
    crn: common determinizations across actions; informed: order-aware playout
    policy (dvc_rollout_batch_flags_ex)."""
    a, ap = _codes(actions)
    P = state.players
    hist = np.zeros((len(a), P), dtype=np.uint64)
    hp = hist.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))
    flags = _flags(crn, informed)
    if flags:
        _check(lib().dvc_rollout_batch_flags_ex(ctypes.byref(state._s), ap, len(a), seed, node_id, sim_begin,
                                                sim_end, flags, hp, device))
    else:
        _check(lib().dvc_rollout_batch_ex(ctypes.byref(state._s), ap, len(a), seed, node_id, sim_begin, sim_end,
                                          hp, None, device))
    return hist


def rollout_batch_fixed_ex(state, actions, rhos, seed, node_id, sim_begin, sim_end, device=-1):
    """The md ablation batch (dvc_rollout_batch_fixed_ex):
    hist[i, w] (numpy uint64) for child i = (determinization rhos[i],
    action actions[i]) over sims [sim_begin, sim_end) (blocking)."""
    a, ap = _codes(actions)
    r = np.ascontiguousarray(np.asarray(rhos, dtype=np.uint64))
    if len(r) != len(a):
        raise ValueError("one rho per action")
    hist = np.zeros((len(a), state.players), dtype=np.uint64)
    _check(lib().dvc_rollout_batch_fixed_ex(ctypes.byref(state._s), ap, r.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                            len(a), seed, node_id, sim_begin, sim_end,
                                            hist.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), device))
    return hist


def sample_determinizations(state, seed, node_id, sim_begin, k):
    """SPEC:230 sample_determinization: the Det(O) indices (canonical order)
    that sims [sim_begin, sim_begin + k) of a CRN batch play (numpy uint64)."""
    out = np.zeros(k, dtype=np.uint64)
    _check(lib().dvc_sample_determinizations(ctypes.byref(state._s), seed, node_id, sim_begin, k,
                                             out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))))
    return out


def md_search(state, n_det, expansions, sims_per_child, seed, c=2 ** 0.5, device=-1):
    """The md ablation search (dvc_md_search).  Returns
    (best_code, [(code, visits, wins)] in LEGAL order, #candidate determinizations)."""
    p = _MdParams(c=c, n_det=n_det, expansions=expansions, sims_per_child=sims_per_child, seed=seed, device=device)
    n = ctypes.c_int32()
    best = ctypes.c_uint32()
    kd = ctypes.c_int32()
    cap = max(1, state.info["n_legal"])
    tab = (_ActionStat * cap)()
    _check(lib().dvc_md_search(ctypes.byref(state._s), ctypes.byref(p), tab, cap, ctypes.byref(n),
                               ctypes.byref(best), ctypes.byref(kd)))
    return best.value, [(t.code, t.visits, t.wins) for t in tab[:n.value]], kd.value


def rollout_path_ex(state, path, actions, seed, node_id, sim_begin, sim_end, device=-1):
    """Deep-tree batch (dvc_rollout_path_ex): returns (hist[A, P], voids[A])."""
    a, ap = _codes(actions)
    p, pp = _codes(path if len(path) else [0])
    P = state.players
    hist = np.zeros((len(a), P), dtype=np.uint64)
    voids = np.zeros(len(a), dtype=np.uint64)
    _check(lib().dvc_rollout_path_ex(ctypes.byref(state._s), pp, len(path), ap, len(a), seed, node_id, sim_begin,
                                     sim_end, hist.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                     voids.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), device))
    return hist, voids


def _stream_ptr(stream, device=None):
    """The launch stream: `stream`, else torch's current stream OF THE DEVICE
    the output tensor lives on (not of the caller's current device)."""
    if stream is None:
        import torch
        stream = torch.cuda.current_stream(device)
    return ctypes.c_void_p(stream.cuda_stream)


def _check_out(t, shape, dtype_name, what):
    """A device output the kernels write with atomics: CUDA, the right dtype,
    shape and contiguous -- anything else would be written out of bounds."""
    import torch
    want = {"int64": torch.int64, "uint8": torch.uint8}[dtype_name]
    if not (isinstance(t, torch.Tensor) and t.is_cuda):
        raise ValueError("%s must be a CUDA tensor" % what)
    if t.dtype != want or tuple(t.shape) != tuple(shape) or not t.is_contiguous():
        raise ValueError("%s must be a contiguous %s tensor of shape %s (got %s %s%s)"
                         % (what, dtype_name, tuple(shape), t.dtype, tuple(t.shape),
                            "" if t.is_contiguous() else ", non-contiguous"))


def rollout_batch_async(state, actions, seed, node_id, sim_begin, sim_end, hist, visits=None, stream=None,
                        crn=False, informed=False):
    """ADD counts into device tensors hist[A, P] (torch.int64, CUDA) and
    visits[A] (optional) on `stream` (default: torch's current stream).
    crn / informed: batch variants (dvc_rollout_batch_flags_async; visits
    must then be None)."""
    a, ap = _codes(actions)
    _check_out(hist, (len(a), state.players), "int64", "hist")
    if visits is not None:
        _check_out(visits, (len(a),), "int64", "visits")
        if visits.device != hist.device:
            raise ValueError("hist and visits must be on the same device")
    dev = hist.device.index
    flags = _flags(crn, informed)
    if flags:
        if visits is not None:
            raise ValueError("the flags entry point takes no visits array")
        _check(lib().dvc_rollout_batch_flags_async(ctypes.byref(state._s), ap, len(a), seed, node_id, sim_begin,
                                                   sim_end, flags, ctypes.c_void_p(hist.data_ptr()), dev,
                                                   _stream_ptr(stream, hist.device)))
        return
    _check(lib().dvc_rollout_batch_async(ctypes.byref(state._s), ap, len(a), seed, node_id, sim_begin, sim_end,
                                         ctypes.c_void_p(hist.data_ptr()),
                                         ctypes.c_void_p(visits.data_ptr()) if visits is not None else None,
                                         dev, _stream_ptr(stream, hist.device)))


def rollout_trace_async(state, actions, seed, node_id, sim_begin, sim_end, hist, winners, stream=None):
    """As rollout_batch_async, plus winners[a*(sim_end-sim_begin) + s - sim_begin]
    (torch.uint8, CUDA) for every playout."""
    a, ap = _codes(actions)
    _check_out(hist, (len(a), state.players), "int64", "hist")
    _check_out(winners, (len(a) * (sim_end - sim_begin),), "uint8", "winners")
    dev = hist.device.index
    _check(lib().dvc_rollout_trace_async(ctypes.byref(state._s), ap, len(a), seed, node_id, sim_begin, sim_end,
                                         ctypes.c_void_p(hist.data_ptr()), ctypes.c_void_p(winners.data_ptr()),
                                         dev, _stream_ptr(stream, hist.device)))


def mcts_search(state, expansions, sims_per_child, seed, c=2 ** 0.5, max_depth=4, flat=1, device=-1, crn=False,
                informed=False):
    """Host UCT over GPU rollout batches (dvc_mcts_search).  Returns
    (best_code, [(code, visits, wins)] in LEGAL order).  crn / informed:
    batch variants for every playout batch (flat = 1 only)."""
    p = _SearchParams(c=c, max_depth=max_depth, expansions=expansions, sims_per_child=sims_per_child,
                      seed=seed, flat=flat, device=device, flags=_flags(crn, informed))
    n = ctypes.c_int32()
    best = ctypes.c_uint32()
    cap = max(1, state.info["n_legal"])
    tab = (_ActionStat * cap)()
    _check(lib().dvc_mcts_search(ctypes.byref(state._s), ctypes.byref(p), tab, cap, ctypes.byref(n),
                                 ctypes.byref(best)))
    return best.value, [(t.code, t.visits, t.wins) for t in tab[:n.value]]


def mcts_search_cb(state, batch, expansions, sims_per_child, seed, c=2 ** 0.5, max_depth=4, flat=1, crn=False,
                   informed=False):
    """dvc_mcts_search_cb: the library's UCT search with every rollout batch
    delegated to batch(path, actions, seed, node_id, sim_begin, sim_end,
    flags) -> (hist [A, P], voids [A] or None), e.g. a sharded + all-reduced
    batch (dist.mcts_search).  Returns (best_code, [(code, visits, wins)])."""
    P = state.players
    err = []

    def _fn(ctx, path, path_len, actions, n_actions, seed_, node_id, s0, s1, flags, hist, voids):
        try:
            h, v = batch([path[i] for i in range(path_len)], [actions[i] for i in range(n_actions)], seed_,
                         node_id, s0, s1, flags)
            h = np.asarray(h, dtype=np.uint64).reshape(-1)
            if h.size != n_actions * P:
                raise ValueError("batch callback returned %d counts for %d x %d" % (h.size, n_actions, P))
            ctypes.memmove(hist, h.ctypes.data, h.nbytes)
            if voids:
                vv = np.zeros(n_actions, dtype=np.uint64) if v is None else np.asarray(v, dtype=np.uint64)
                ctypes.memmove(voids, vv.ctypes.data, vv.nbytes)
            return 0
        except DvcError as e:
            err.append(e)
            return e.code
        except Exception as e:  # surfaced below; the C side sees a failure code
            err.append(e)
            return -1

    cb = BATCH_FN(_fn)
    p = _SearchParams(c=c, max_depth=max_depth, expansions=expansions, sims_per_child=sims_per_child,
                      seed=seed, flat=flat, device=-1, flags=_flags(crn, informed))
    n = ctypes.c_int32()
    best = ctypes.c_uint32()
    cap = max(1, state.info["n_legal"])
    tab = (_ActionStat * cap)()
    rc = lib().dvc_mcts_search_cb(ctypes.byref(state._s), ctypes.byref(p), cb, None, tab, cap, ctypes.byref(n),
                                  ctypes.byref(best))
    if err:
        raise err[0]
    _check(rc)
    return best.value, [(t.code, t.visits, t.wins) for t in tab[:n.value]]


def set_option(name, value):
    _check(lib().dvc_set_option(name.encode(), int(value)))


def get_option(name):
    v = ctypes.c_int64()
    _check(lib().dvc_get_option(name.encode(), ctypes.byref(v)))
    return v.value


class options:
    """Context manager: temporarily set launch options (they never change results)."""

    def __init__(self, **kw):
        self.kw = kw
        self.old = {}

    def __enter__(self):
        for k, v in self.kw.items():
            self.old[k] = get_option(k)
            set_option(k, v)
        return self

    def __exit__(self, *exc):
        for k, v in self.old.items():
            set_option(k, v)


def debug_counters(device=-1):
    """(violations, first code, playouts checked) -- debug build only."""
    out = (ctypes.c_uint32 * 3)()
    _check(lib().dvc_debug_counters(device, out))
    return tuple(out)


def launch_count(reset=False):
    return int(lib().dvc_launch_count(1 if reset else 0))


def transfer_bytes(reset=False):
    """(host->device, device->host) bytes the library moved since the last
    reset (dvc_transfer_bytes): copies plus kernel parameter blocks."""
    h, d = ctypes.c_uint64(), ctypes.c_uint64()
    _check(lib().dvc_transfer_bytes(1 if reset else 0, ctypes.byref(h), ctypes.byref(d)))
    return int(h.value), int(d.value)


def shutdown():
    lib().dvc_shutdown()
