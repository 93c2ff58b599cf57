"""Layer-wise DA / DBA plan (the reference's ``LayerPlan`` /
``plan_layers``, /root/reference/pkg/src/offsim/pipeline.py:177-195).

The reference picks, per layer, the batch-split schedule (``"dba"``) wherever that
layer's mean miss count per request-step reaches a threshold theta, and the plain
overlap (``"da"``) elsewhere; the simulator then prices each layer with its own span
DAG.  Here the plan drives the real schedule: ``DSADecodeModel.capture(plan=...)``
records every layer with its own strategy into the one step graph (DBA layers
micro-batched K1-K3 under the gather, DA layers one batch with the fused K5).

The miss means come from either
  * a ``MissProfile`` (``cache.replay`` of an ESSTRACE, the reference's input), or
  * the model's own pools: ``MissMeter`` differences the per-pool miss counters
    (cache.py:41-43) over the steps since its snapshot — the running mean of the
    live decode, with no host sync inside the step.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

STRATEGIES = ("none", "da", "dba")


@dataclass
class LayerPlan:
    """pipeline.py:177-187: one strategy tag per layer, the threshold it came from."""
    strategies: list[str]
    threshold: float
    source: str = ""

    def counts(self) -> dict[str, int]:
        out: dict[str, int] = {}
        for tag in self.strategies:
            out[tag] = out.get(tag, 0) + 1
        return out

    def check(self, num_layers: int) -> None:
        if len(self.strategies) != num_layers:
            raise ValueError(f"plan has {len(self.strategies)} strategies for {num_layers} layers")
        bad = [s for s in self.strategies if s not in STRATEGIES]
        if bad:
            raise ValueError(f"unknown strategies in plan: {sorted(set(bad))}")


def plan_from_means(means, threshold: float, source: str = "") -> LayerPlan:
    """pipeline.py:190-195: ``dba`` where the layer's mean misses >= threshold, else ``da``."""
    means = np.asarray(means, dtype=np.float64)
    return LayerPlan(strategies=["dba" if m >= threshold else "da" for m in means],
                     threshold=float(threshold), source=source)


def plan_layers(profile, threshold: float, source: str = "") -> LayerPlan:
    """The reference's entry point: a plan from a ``MissProfile`` (misses[L, T] of one
    request's replay; ``layer_means`` = mean over steps)."""
    return plan_from_means(profile.layer_means(), threshold, source)


class MissMeter:
    """Running per-layer miss means of a decode model from its pools' own counters.

    ``snapshot()`` records every layer's (requests, misses) totals; ``means()`` is, per
    layer, the misses since the snapshot divided by request-steps since the snapshot —
    the live analogue of ``MissProfile.layer_means`` (one request's misses per layer per
    step), averaged over the layer's requests."""

    def __init__(self, model):
        self.model = model
        self.snapshot()

    def _totals(self):
        return np.array([layer.access_totals()[1] for layer in self.model.layers], dtype=np.int64)

    def _steps(self):
        return np.array([layer.history for layer in self.model.layers], dtype=np.int64)

    def snapshot(self) -> None:
        self._m0, self._t0 = self._totals(), self._steps()

    def means(self) -> np.ndarray:
        steps = self._steps() - self._t0
        if (steps <= 0).any():
            raise ValueError("no decode step since the miss meter's snapshot")
        return (self._totals() - self._m0) / (steps * self.model.B)
