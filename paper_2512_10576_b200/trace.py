"""Selection traces: the top-k output contract and the synthetic workload.

Host-side tooling (no device code).  Mirrors the reference's trace module
surface (/root/reference/pkg/src/offsim/trace.py):

* ``StepAccess`` / ``AccessTrace`` (trace.py:31-65): per (step, layer) a strictly
  increasing uint32 id set — exactly what the top-k kernel emits.
* ``TraceGenParams`` / ``generate_trace`` (trace.py:68-161): the retention +
  Gumbel-top-k generator.  Restated so that, for the same numpy version, the
  random stream and therefore every selection set is identical to the
  reference's (checked against committed fixtures in tests/golden/).
* ``ESSTRACE`` v1 binary I/O (trace.py:199-287) with byte-offset
  errors, and Eq. (1) similarity (trace.py:164-196).

The generator is the bench's trace-driven workload; it never runs inside a
timed region.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np

TRACE_MAGIC = b"ESSTRACE"
TRACE_VERSION = 1
PREFILL_WINDOW_COUNT = 32
_HEADER = struct.Struct("<HIQIQB")


class TraceFormatError(ValueError):
    """Malformed trace bytes; ``offset`` is where the fault was detected."""

    def __init__(self, message: str, offset: int):
        super().__init__(f"{message} (byte offset {offset})")
        self.offset = offset


@dataclass
class StepAccess:
    layers: list
    tokens_accepted: int = 1


@dataclass
class AccessTrace:
    num_layers: int
    context_len: int
    topk: int
    steps: list
    prefill_windows: list | None = None

    @property
    def num_steps(self) -> int:
        return len(self.steps)

    def tokens_generated_before(self, step: int) -> int:
        return int(sum(s.tokens_accepted for s in self.steps[:step]))

    def check(self) -> None:
        """ValueError on any layer-count, ordering or range violation (trace.py:55-65)."""
        limit = self.context_len
        for t, step in enumerate(self.steps):
            if len(step.layers) != self.num_layers:
                raise ValueError(
                    f"step {t}: expected {self.num_layers} layers, got {len(step.layers)}")
            for l, ids in enumerate(step.layers):
                a = np.asarray(ids, dtype=np.int64)
                if a.size and np.any(a[1:] <= a[:-1]):
                    raise ValueError(f"step {t} layer {l}: indices not strictly increasing")
                if a.size and (a[0] < 0 or a[-1] >= limit):
                    raise ValueError(f"step {t} layer {l}: index out of range [0, {limit})")
            limit += step.tokens_accepted

    def padded_step(self, t: int, width: int | None = None):
        """(ids [L, width] int32 padded with -1, counts [L] int32) for device upload."""
        layers = self.steps[t].layers
        width = width or max(1, max(len(a) for a in layers))
        out = np.full((self.num_layers, width), -1, np.int32)
        n = np.zeros(self.num_layers, np.int32)
        for l, a in enumerate(layers):
            out[l, :len(a)] = a
            n[l] = len(a)
        return out, n


@dataclass
class TraceGenParams:
    num_layers: int = 4
    context_len: int = 32768
    topk: int = 2048
    num_steps: int = 100
    target_similarity: float = 0.9
    recency_bias: float = 1.0
    mean_accept: float = 1.7
    layer_similarity_overrides: dict = field(default_factory=dict)
    seed: int = 0

    def violations(self) -> list:
        bad = []
        if not 0.0 <= self.target_similarity <= 1.0:
            bad.append("target_similarity must be in [0, 1]")
        bad += [f"layer {l} similarity override must be in [0, 1]"
                for l, r in self.layer_similarity_overrides.items() if not 0.0 <= r <= 1.0]
        if self.mean_accept < 1.0:
            bad.append("mean_accept must be >= 1")
        if self.topk > self.context_len:
            bad.append("topk must not exceed context_len at step 0")
        if min(self.num_steps, self.num_layers) < 1:
            bad.append("num_steps and num_layers must be >= 1")
        return bad


def _gumbel(rng: np.random.Generator, n: int) -> np.ndarray:
    return -np.log(-np.log(rng.random(n)))


class _RetentionProcess:
    """One layer's selection process (trace.py:96-113 semantics).

    Each event keeps every current member with probability r, then refills to k
    members by Gumbel-top-k over the recency log-weights of the non-members.
    """

    def __init__(self, rng, log_weight, k, r):
        self.rng, self.logw, self.k, self.r = rng, log_weight, k, r
        self.member = np.zeros(len(log_weight), dtype=bool)

    def seed(self, universe: int):
        scores = self.logw[:universe] + _gumbel(self.rng, universe)
        top = np.argpartition(scores, universe - self.k)[universe - self.k:]
        self.member[top] = True

    def advance(self, universe: int):
        cur = np.flatnonzero(self.member[:universe])
        kept = cur[self.rng.random(cur.size) < self.r]
        need = self.k - kept.size
        nxt = np.zeros_like(self.member)
        nxt[kept] = True
        if need > 0:
            free = np.flatnonzero(~nxt[:universe])
            scores = self.logw[free] + _gumbel(self.rng, free.size)
            nxt[free[np.argpartition(scores, free.size - need)[free.size - need:]]] = True
        self.member = nxt

    def snapshot(self) -> np.ndarray:
        return np.flatnonzero(self.member).astype(np.uint32)


def generate_trace(p: TraceGenParams) -> AccessTrace:
    """Deterministic synthetic trace with tunable step-to-step overlap (trace.py:116-161)."""
    bad = p.violations()
    if bad:
        raise ValueError("; ".join(bad))
    rng = np.random.default_rng(p.seed)
    accepted = rng.poisson(p.mean_accept - 1.0, size=p.num_steps).astype(int) + 1
    universe_max = p.context_len + int(accepted.sum())
    logw = p.recency_bias * np.log1p(np.arange(universe_max, dtype=np.float64))

    per_layer, windows = [], []
    for layer in range(p.num_layers):
        proc = _RetentionProcess(np.random.default_rng(np.random.SeedSequence([p.seed, layer])),
                                 logw, p.topk,
                                 p.layer_similarity_overrides.get(layer, p.target_similarity))
        proc.seed(p.context_len)
        wins = [proc.snapshot()]
        for _ in range(PREFILL_WINDOW_COUNT - 1):
            proc.advance(p.context_len)
            wins.append(proc.snapshot())
        windows.append(wins)
        sets, universe = [], p.context_len
        for t in range(p.num_steps):
            proc.advance(universe)
            sets.append(proc.snapshot())
            universe += int(accepted[t])
        per_layer.append(sets)

    steps = [StepAccess([per_layer[l][t] for l in range(p.num_layers)], int(accepted[t]))
             for t in range(p.num_steps)]
    return AccessTrace(p.num_layers, p.context_len, p.topk, steps, windows)


def intra_layer_similarity(trace: AccessTrace, layer: int) -> np.ndarray:
    """|K_{t-1} & K_t| / |K_t| for t >= 1 (Eq. (1); trace.py:164-177)."""
    if not 0 <= layer < trace.num_layers:
        raise ValueError(f"layer {layer} out of range")
    out = np.zeros(max(0, trace.num_steps - 1))
    for t in range(1, trace.num_steps):
        a, b = trace.steps[t - 1].layers[layer], trace.steps[t].layers[layer]
        out[t - 1] = (np.intersect1d(a, b, assume_unique=True).size / len(b)) if len(b) else 0.0
    return out


@dataclass
class LayerSimilarity:
    layer: int
    mean: float
    stdev: float
    min: float


def similarity_summary(trace: AccessTrace) -> list:
    if trace.num_steps < 2:
        raise ValueError("similarity summary needs at least 2 steps")
    res = []
    for l in range(trace.num_layers):
        r = intra_layer_similarity(trace, l)
        res.append(LayerSimilarity(l, float(r.mean()), float(r.std()), float(r.min())))
    return res


# ------------------------------------------------------------------------------------
# ESSTRACE v1 (little endian): magic, <HIQIQB header, per step <H accepted + per layer
# <I count + count delta-coded <u4 (first absolute), optional <I nwin + windows.
# ------------------------------------------------------------------------------------

def _pack_ids(ids) -> bytes:
    a = np.asarray(ids, dtype=np.uint32)
    if a.size == 0:
        return struct.pack("<I", 0)
    d = np.empty_like(a)
    d[0] = a[0]
    d[1:] = a[1:] - a[:-1]
    return struct.pack("<I", a.size) + d.astype("<u4").tobytes()


def encode_trace(trace: AccessTrace) -> bytes:
    parts = [TRACE_MAGIC, _HEADER.pack(TRACE_VERSION, trace.num_layers, trace.context_len,
                                       trace.topk, trace.num_steps,
                                       int(trace.prefill_windows is not None))]
    for st in trace.steps:
        parts.append(struct.pack("<H", st.tokens_accepted))
        parts += [_pack_ids(a) for a in st.layers]
    if trace.prefill_windows is not None:
        parts.append(struct.pack("<I", len(trace.prefill_windows[0]) if trace.prefill_windows else 0))
        for wins in trace.prefill_windows:
            parts += [_pack_ids(w) for w in wins]
    return b"".join(parts)


def write_trace(trace: AccessTrace, path) -> None:
    with open(path, "wb") as f:
        f.write(encode_trace(trace))


class _Cursor:
    def __init__(self, buf: bytes):
        self.buf, self.at = buf, 0

    def bytes(self, n: int, what: str) -> bytes:
        if self.at + n > len(self.buf):
            raise TraceFormatError(f"truncated file while reading {what}", self.at)
        b = self.buf[self.at:self.at + n]
        self.at += n
        return b

    def fmt(self, f: str, what: str):
        return struct.unpack(f, self.bytes(struct.calcsize(f), what))

    def ids(self, limit: int, what: str) -> np.ndarray:
        start = self.at
        (n,) = self.fmt("<I", f"{what} count")
        d = np.frombuffer(self.bytes(4 * n, f"{what} indices"), dtype="<u4")
        if n and np.any(d[1:] == 0):
            raise TraceFormatError(f"{what}: duplicate index (zero delta)", start)
        v = np.cumsum(d, dtype=np.uint64)
        if n and int(v[-1]) >= limit:
            raise TraceFormatError(f"{what}: index {int(v[-1])} out of range [0, {limit})", start)
        return v.astype(np.uint32)


def decode_trace(buf: bytes) -> AccessTrace:
    c = _Cursor(buf)
    if c.bytes(len(TRACE_MAGIC), "magic") != TRACE_MAGIC:
        raise TraceFormatError(f"bad magic {buf[:len(TRACE_MAGIC)]!r}, expected {TRACE_MAGIC!r}", 0)
    ver, L, ctx, topk, T, has_win = c.fmt(_HEADER.format, "header")
    if ver != TRACE_VERSION:
        raise TraceFormatError(f"unsupported version {ver}", len(TRACE_MAGIC))
    steps, gen = [], 0
    for t in range(T):
        (acc,) = c.fmt("<H", f"step {t} tokens_accepted")
        steps.append(StepAccess([c.ids(ctx + gen, f"step {t} layer {l}") for l in range(L)], acc))
        gen += acc
    windows = None
    if has_win:
        (nw,) = c.fmt("<I", "prefill window count")
        windows = [[c.ids(ctx, f"prefill layer {l} window {w}") for w in range(nw)]
                   for l in range(L)]
    if c.at != len(buf):
        raise TraceFormatError("trailing bytes after trace body", c.at)
    return AccessTrace(L, ctx, topk, steps, windows)


def read_trace(path) -> AccessTrace:
    with open(path, "rb") as f:
        return decode_trace(f.read())
