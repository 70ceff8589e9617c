"""GPU: the bench contract end to end (bench.py is what the driver runs).

One GPU runs `python bench.py`, `torchrun --nproc-per-node 1 bench.py` and --
as a FUNCTIONAL test of the N > 1 code path only, never a measurement --
`torchrun --nproc-per-node 2` with BENCH_BACKEND=gloo (two ranks share the one
GPU; the all_reduces go through host copies).  Every line must carry the
contract's keys, merge_bit_exact (rank 0's recomputation of the merged range)
and the C4 strong-scaling record, whose merged histogram (sha256) must be the
same at N = 1 and N = 2 (keyed Philox + integer sums: bit-identical at any N)."""

import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

ARGS = ["--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--no-deals", "--sims", "200000"]
KEYS = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks", "merge_bit_exact",
        "c4_strong"]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(cmd, env=None):
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900,
                         env=dict(os.environ, **(env or {})))
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]          # rank 0 alone prints ONE line
    return json.loads(lines[0])


def _check(line, n):
    for k in KEYS:
        assert k in line, k
    assert line["n_gpus"] == n and line["value"] > 0 and line["gpu_launches"] > 0
    assert line["merge_bit_exact"] is True
    c4 = line["c4_strong"]
    assert c4["merge_bit_exact"] is True and c4["playouts_per_move"] >= 10 ** 8
    r = line["roofline"]
    assert r["bound"] == "alu" and 0 < r["frac"] < 1 and 0 < r["frac_fixed_unit"] < 1
    e = line["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0


def test_bench_line_n1_and_torchrun():
    a = _run([sys.executable, "bench.py"] + ARGS)
    _check(a, 1)
    tr = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--master-addr", "127.0.0.1"]
    b = _run(tr + ["--nproc-per-node", "1", "--master-port", str(_port()), "bench.py", "--gpus", "1"] + ARGS)
    _check(b, 1)
    c = _run(tr + ["--nproc-per-node", "2", "--master-port", str(_port()), "bench.py", "--gpus", "2"] + ARGS,
             env={"BENCH_BACKEND": "gloo"})
    _check(c, 2)
    assert a["c4_strong"]["hist_sha256"] == b["c4_strong"]["hist_sha256"] == c["c4_strong"]["hist_sha256"]
