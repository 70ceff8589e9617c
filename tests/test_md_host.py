"""Host-side (no GPU) pins of the md ablation's boundary:
dvc_sample_determinizations equals the oracle's CRN
determinization ranks, and the md entry points validate their arguments."""

import glob
import json
import os

import pytest

from conftest import ROOT
from oracle import philox as px


@pytest.fixture(scope="module")
def dvc():
    from paper_2403_10720_b200 import build
    build.build()
    from paper_2403_10720_b200 import dvc as m
    return m


@pytest.mark.parametrize("name", ["c1_d1", "c2_d1", "c3_d1", "c4_d2", "x3_d1"])
def test_sample_determinizations_equal_oracle(dvc, oracle_lib, name):
    d = json.load(open(os.path.join(ROOT, "fixtures", name + ".json")))
    st = dvc.encode(d)
    N = oracle_lib.count(d)
    for seed, node, s0 in ((1, 0, 0), (0xDEADBEEF12345678, 77, 4000), (5, 0xFFFFFFFF, (1 << 32) - 50)):
        got = dvc.sample_determinizations(st, seed, node, s0, 50).tolist()
        exp = [px.rank64(N, *px.det_block(seed, node, px.CRN_WORD, s0 + i)) for i in range(50)]
        assert got == exp


def test_sample_determinizations_errors(dvc):
    d = json.load(open(os.path.join(ROOT, "fixtures", "c2_d1.json")))
    st = dvc.encode(d)
    with pytest.raises(dvc.DvcError):
        dvc.sample_determinizations(st, 1, 0, (1 << 32) - 10, 11)      # past the 32-bit sim range
    assert len(dvc.sample_determinizations(st, 1, 0, 0, 0)) == 0


def test_md_search_argument_errors(dvc):
    d = json.load(open(os.path.join(ROOT, "fixtures", "c2_d1.json")))
    st = dvc.encode(d)
    for bad in (dict(n_det=0), dict(n_det=4097), dict(expansions=0), dict(sims_per_child=0)):
        kw = dict(n_det=4, expansions=8, sims_per_child=8, seed=1)
        kw.update(bad)
        with pytest.raises(dvc.DvcError) as e:
            dvc.md_search(st, **kw)
        assert e.value.code == -1
