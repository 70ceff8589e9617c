"""Host-side tests of the C-ABI boundary (no GPU needed): libdvc.so loads and
exports every symbol include/dvc.h declares; dvc_state_encode's validation
classes (dvc.h); the host encoder's determinization count and
legal-action list equal the oracle's on every fixture; rollout entry points
fail loudly (DVC_E_CUDA) without a device -- there is no CPU fallback."""

import copy
import glob
import json
import os
import re

import pytest

from conftest import ROOT

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def dvc():
    from paper_2403_10720_b200 import build
    build.build()
    from paper_2403_10720_b200 import dvc as m
    return m


def test_exports_every_declared_symbol(dvc):
    hdr = open(os.path.join(ROOT, "include", "dvc.h")).read()
    declared = set(re.findall(r"\b(dvc_[a-z_0-9]+)\s*\(", hdr))
    assert declared == set(dvc.EXPORTS)
    L = dvc.lib()
    for name in declared:
        assert hasattr(L, name), name


ALL = sorted(glob.glob(os.path.join(ROOT, "fixtures", "*.json"))) + \
    sorted(glob.glob(os.path.join(ROOT, "tests", "golden", "*.json")))


@pytest.mark.parametrize("path", ALL, ids=[os.path.basename(p) for p in ALL])
def test_encode_matches_oracle(dvc, oracle_lib, path):
    d = json.load(open(path))
    st = dvc.encode(d)
    info = st.info
    assert info["n_det"] == oracle_lib.count(d)
    legal = st.legal_actions()
    assert legal == oracle_lib.legal(d)
    assert info["n_legal"] == len(legal)
    assert info["viewer"] == d["viewer"]
    # pointer-free POD: round-trips through bytes
    st2 = dvc.State.from_bytes(st.to_bytes())
    assert st2.legal_actions() == legal


def _base():
    return json.load(open(os.path.join(ROOT, "tests", "golden", "T2c1.json")))


def _err(dvc, d):
    with pytest.raises(dvc.DvcError) as e:
        dvc.encode(d)
    return e.value.code


def test_encode_errors(dvc):
    d = _base()
    bad = copy.deepcopy(d); bad["rules"]["players"] = 5
    assert _err(dvc, bad) == -1
    bad = copy.deepcopy(d); bad["rules"]["ranks"] = 13
    assert _err(dvc, bad) == -1
    bad = copy.deepcopy(d); bad["lines"][0][1] = {"color": "B", "value": 0, "revealed": False}   # B0 twice
    assert _err(dvc, bad) == -4
    bad = copy.deepcopy(d); bad["pool_size"] = 3                                                  # conservation
    assert _err(dvc, bad) == -4
    bad = copy.deepcopy(d); bad["lines"][0] = [d["lines"][0][1], d["lines"][0][0]]               # unsorted
    bad["pending"] = 0
    assert _err(dvc, bad) == -4
    bad = copy.deepcopy(d); bad["lines"][1][0]["value"] = 1                                       # valued hidden
    assert _err(dvc, bad) == -4
    bad = copy.deepcopy(d); bad["pending"] = -1                                                   # no draw
    assert _err(dvc, bad) == -2
    bad = copy.deepcopy(d); bad["correct_this_turn"] = 1; bad["rules"]["consecutive"] = 0
    assert _err(dvc, bad) == -2
    bad = copy.deepcopy(d); bad["lines"][0][0]["revealed"] = True; bad["lines"][0][1]["revealed"] = True
    assert _err(dvc, bad) == -2                                                                   # viewer dead


def test_e3_inconsistent_when_no_determinization(dvc):
    d = json.load(open(os.path.join(ROOT, "tests", "golden", "E3.json")))
    bad = copy.deepcopy(d)
    # opponent [B?, W0 revealed] but the viewer now owns B0: nothing fits left of W0
    bad["lines"][0] = [{"color": "B", "value": 0, "revealed": True}, {"color": "W", "value": 2, "revealed": False}]
    assert _err(dvc, bad) == -4


@pytest.mark.skipif(torch.cuda.is_available(), reason="CPU-only check")
def test_rollout_without_gpu_fails_loudly(dvc):
    d = _base()
    st = dvc.encode(d)
    codes = st.legal_actions()
    with pytest.raises(dvc.DvcError) as e:
        dvc.rollout_batch(st, codes, 10, 1)
    assert e.value.code == -6
    with pytest.raises(dvc.DvcError) as e:
        dvc.rollout_batch(st, [0x01000000 | 5], 10, 1)     # W2 is the viewer's own: illegal
    assert e.value.code == -3
    with pytest.raises(dvc.DvcError) as e:
        dvc.rollout_batch(st, codes, 0, 1)
    assert e.value.code == -1
    with pytest.raises(dvc.DvcError) as e:
        dvc.rollout_batch(st, [], 10, 1)                     # empty action list
    assert e.value.code == -1
    with pytest.raises(dvc.DvcError) as e:
        dvc.rollout_batch(st, codes * 400, 10, 1)            # more than 768 actions
    assert e.value.code == -1
    with pytest.raises(dvc.DvcError) as e:
        dvc.rollout_batch(st, codes, 1 << 32, 1)             # sim indices are 32-bit
    assert e.value.code == -1


def test_options_roundtrip(dvc):
    old = dvc.get_option("block")
    with dvc.options(block=128, kernel=1):
        assert dvc.get_option("block") == 128 and dvc.get_option("kernel") == 1
    assert dvc.get_option("block") == old and dvc.get_option("kernel") == 2   # auto
    with pytest.raises(dvc.DvcError):
        dvc.set_option("block", 1025)
    with pytest.raises(dvc.DvcError):
        dvc.set_option("kernel", 3)
    with pytest.raises(dvc.DvcError):
        dvc.set_option("nope", 1)
    assert dvc.get_option("search_device") == 0            # host tree by default (north_star)
    with dvc.options(search_device=1):
        assert dvc.get_option("search_device") == 1
    with pytest.raises(dvc.DvcError):
        dvc.set_option("search_device", 2)


def test_every_export_has_argtypes(dvc):
    """Every C-ABI entry point the binding uses declares its argument types
    (ctypes would otherwise pass 64-bit arguments as C ints)."""
    L = dvc.lib()
    for name in dvc.EXPORTS:
        if name in ("dvc_last_error", "dvc_shutdown"):
            continue
        assert getattr(L, name).argtypes is not None, name
