"""Device-side rule invariants (SURVEY §8(c.8) "Rules" row, asserted in the
GPU debug build): libdvc_debug.so checks, after every decision step of every
playout, tile conservation, revealed tiles held, valid joker thresholds, a
live mover, one reveal per guess, STOP only after a correct guess, the
decision bound and a single survivor.  Run over every fixture, both kernels,
plain and deep-tree batches; zero violations allowed."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]


def test_device_invariants_hold():
    from paper_2403_10720_b200 import build
    build.build(debug=True)
    env = dict(os.environ, DVC_DEBUG="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "debug_invariants_run.py"), "20000"],
                         env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    violations, first, checked = res["counters"]
    assert checked > 1000000
    assert violations == 0, "first violation code %d" % first
