"""Layer-wise DA/DBA plan: the host logic of plan.py against the
reference's plan_layers (pipeline.py:190-195) on the same miss profiles."""
from __future__ import annotations

import os
import sys

import numpy as np
import pytest

from paper_2512_10576_b200.cache import MissProfile
from paper_2512_10576_b200.plan import LayerPlan, plan_from_means, plan_layers

REF = "/root/reference/pkg/src"


def _profiles():
    rng = np.random.default_rng(5)
    for L, T in [(1, 1), (3, 4), (61, 16)]:
        yield MissProfile(misses=rng.integers(0, 400, size=(L, T)).astype(np.int64), sparse_ratio=0.25)
    yield MissProfile(misses=np.full((4, 3), 120, np.int64), sparse_ratio=0.1)  # ties at theta


@pytest.mark.parametrize("theta", [0.0, 100.0, 120.0, 200.0, 1e9])
def test_plan_layers_threshold_rule(theta):
    for prof in _profiles():
        plan = plan_layers(prof, theta, source="t")
        means = prof.misses.mean(axis=1)
        assert plan.strategies == ["dba" if m >= theta else "da" for m in means]
        assert sum(plan.counts().values()) == prof.num_layers
        assert plan.threshold == theta and plan.source == "t"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference checkout not present")
@pytest.mark.parametrize("theta", [0.0, 120.0, 250.0])
def test_plan_layers_equals_reference(theta):
    sys.path.insert(0, REF)
    try:
        from offsim.cache import MissProfile as RefProfile
        from offsim.pipeline import plan_layers as ref_plan
    finally:
        sys.path.remove(REF)
    for prof in _profiles():
        ref = ref_plan(RefProfile(misses=prof.misses, sparse_ratio=prof.sparse_ratio), theta, "s")
        ours = plan_layers(prof, theta, "s")
        assert ours.strategies == ref.strategies and ours.counts() == ref.counts()


def test_plan_check_rejects_bad_plans():
    with pytest.raises(ValueError):
        LayerPlan(["da", "dba"], 1.0).check(3)
    with pytest.raises(ValueError):
        LayerPlan(["da", "tbo"], 1.0).check(2)
    plan_from_means([1.0, 2.0], 1.5).check(2)
