"""The device pass's scheduling variants must not change a single bit: the full 10k-search
batch (1 MiB buckets) with the default schedule, with every layer step through the
two-kernel path (K2a + K2b, no K2t), with every step through the one-kernel path (K2t), and
with one sweep after all bands instead of per-band sweeps.  The knobs are read once per
process, so each variant runs in its own subprocess and reports a digest of its results and
plans.  Needs a B200 (-m gpu)."""

from __future__ import annotations

import hashlib
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

_SCRIPT = r"""
import hashlib, sys
sys.path.insert(0, {root!r})
import numpy as np
from paper_2307_02031_b200 import workloads as W
from paper_2307_02031_b200.dpsearch import run_native_batch
L, S, E, P, T = W.sweep_arrays(W.sweep_cells(10_000))
rc, msg, res, plans, _ = run_native_batch(L, S, E, P, None)
assert rc == 0, msg
h = hashlib.sha256()
for f in ("feasible", "time_s", "e_fwd", "stage_time", "stage_ns", "stage_peak"):
    h.update(np.ascontiguousarray(res[f]).tobytes())
h.update(plans.tobytes())
print("DIGEST", h.hexdigest(), int(res["feasible"].sum()))
"""


def _digest(env_extra):
    env = dict(os.environ)
    env.update(env_extra)
    out = subprocess.run([sys.executable, "-c", _SCRIPT.format(root=str(ROOT))], env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    line = [x for x in out.stdout.splitlines() if x.startswith("DIGEST")][-1]
    _, digest, feasible = line.split()
    return digest, int(feasible)


def test_schedule_variants_bit_identical(gpu):
    base = _digest({})
    assert base[1] > 0
    for extra in ({"GBMW_TILE_FUSED_MAX": "0"}, {"GBMW_TILE_FUSED_MAX": "1000000000"},
                  {"GBMW_SWEEP_PER_GROUP": "0"}):
        assert _digest(extra) == base, extra
