"""§8f.4 live selections -> ESSTRACE: a trace recorded from the GPU decode step (C1
shape, committed fixture from scripts/export_live_trace.py) is a valid reference
trace, and replaying it through the reference's LRU (our C restatement here; the
reference itself when importable) reproduces the miss counts the device cache
manager reported during the run."""
import json
import os
import sys

import numpy as np
import pytest

from oracle import lru as olru
from paper_2512_10576_b200 import trace as etrace

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIX = os.path.join(ROOT, "tests", "golden", "live_c1")
OFFSIM = "/root/reference/pkg/src"


def _fixture():
    tr = etrace.read_trace(FIX + ".esstrace")
    with open(FIX + ".json") as f:
        meta = json.load(f)
    return tr, meta


def test_live_trace_round_trips_and_is_canonical():
    tr, _ = _fixture()
    tr.check()
    assert tr.num_layers == 1 and tr.topk == 2048 and tr.prefill_windows is not None
    raw = etrace.encode_trace(tr)
    assert etrace.encode_trace(etrace.decode_trace(raw)) == raw
    sims = etrace.similarity_summary(tr)
    assert 0.5 < sims[0].mean <= 1.0          # drifting queries: high step-to-step overlap


def test_oracle_replay_of_live_trace_matches_device_misses():
    tr, meta = _fixture()
    steps = [s.layers for s in tr.steps]
    got = olru.replay_misses(steps, [s.tokens_accepted for s in tr.steps], tr.context_len,
                             meta["sparse_ratio"], windows=tr.prefill_windows, use_warmup=True)
    np.testing.assert_array_equal(got[0], meta["device_misses_per_step"])


@pytest.mark.skipif(not os.path.isdir(OFFSIM), reason="reference not present (GPU box)")
def test_reference_reads_and_replays_live_trace():
    sys.path.insert(0, OFFSIM)
    try:
        from offsim import cache as rcache
        from offsim import trace as rtrace
    finally:
        sys.path.remove(OFFSIM)
    _, meta = _fixture()
    tr = rtrace.read_trace(FIX + ".esstrace")
    prof = rcache.replay(tr, meta["sparse_ratio"], use_warmup=True)
    np.testing.assert_array_equal(np.asarray(prof.misses)[0], meta["device_misses_per_step"])
    assert rtrace.similarity_summary(tr)[0].mean > 0.5
