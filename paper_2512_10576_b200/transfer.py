"""Host latent store and the zero-copy miss gather (K4).

* ``TransferModel`` / ``transfer_time`` restate the reference's PCIe yardstick
  (/root/reference/pkg/src/offsim/costmodel.py:128-186): batched FlashTrans
  37/43 GB/s and per-call cudaMemcpyAsync 0.79/0.23 GB/s at 656-B blocks
  (PAPER.md:273, :279).  The bench reports measured gather GB/s against these.
* ``HostLatentStore`` — the CPU-side "total memory pool": pinned,
  mapped (cudaHostRegister) so the gather kernel reads rows with 16-B loads.
* ``gather`` / ``write_generated`` — the H2D miss fill and the D2H write-back of
  newly generated rows (cache.py:122-134).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

from . import _lib
from .cache import AccessBatch, PoolSet

LATENT_BLOCK_BYTES = 656
# K4 form: 16-B zero-copy loads (False) or cp.async.bulk row copies into a smem ring (True)
GATHER_BULK = os.environ.get("ESS_GATHER_BULK", "0") == "1"
# the host store as one host-located VMM allocation (ess_host_alloc ESS_HOST_VMM)
HOST_VMM = os.environ.get("ESS_HOST_VMM", "0") == "1"
PER_CALL_EFFECTIVE_H2D_GBS = 0.79
PER_CALL_EFFECTIVE_D2H_GBS = 0.23


def fit_per_call_overhead_us(block_bytes: float, bw_link_gbs: float, bw_effective_gbs: float) -> float:
    """Per-copy overhead making a ``bw_link_gbs`` link deliver ``bw_effective_gbs``."""
    return block_bytes * (1.0 / bw_effective_gbs - 1.0 / bw_link_gbs) / 1e3


@dataclass(frozen=True)
class TransferModel:
    mode: str = "batched"
    bw_h2d_gbs: float = 37.0
    bw_d2h_gbs: float = 43.0
    block_bytes: int = LATENT_BLOCK_BYTES
    per_call_overhead_h2d_us: float | None = None
    per_call_overhead_d2h_us: float | None = None

    def __post_init__(self):
        if self.mode not in ("per_call", "batched"):
            raise ValueError(f"unknown transfer mode {self.mode!r}")
        if min(self.bw_h2d_gbs, self.bw_d2h_gbs) <= 0:
            raise ValueError("bandwidths must be > 0")
        for attr, bw, eff in (("per_call_overhead_h2d_us", self.bw_h2d_gbs, PER_CALL_EFFECTIVE_H2D_GBS),
                              ("per_call_overhead_d2h_us", self.bw_d2h_gbs, PER_CALL_EFFECTIVE_D2H_GBS)):
            if getattr(self, attr) is None:
                object.__setattr__(self, attr, fit_per_call_overhead_us(self.block_bytes, bw, eff))
        if min(self.per_call_overhead_h2d_us, self.per_call_overhead_d2h_us) < 0:
            raise ValueError("per-call overheads must be >= 0")


def transfer_time(model: TransferModel, blocks: int, direction: str) -> float:
    """Microseconds to move ``blocks`` latent rows one way (costmodel.py:173-186)."""
    if blocks < 0:
        raise ValueError("blocks must be >= 0")
    if direction not in ("h2d", "d2h"):
        raise ValueError(f"direction must be h2d or d2h, got {direction!r}")
    h2d = direction == "h2d"
    us = blocks * model.block_bytes / ((model.bw_h2d_gbs if h2d else model.bw_d2h_gbs) * 1e3)
    if model.mode == "per_call":
        us += blocks * (model.per_call_overhead_h2d_us if h2d else model.per_call_overhead_d2h_us)
    return us


def gpu_numa_node(device=None) -> int | None:
    """NUMA node of the GPU's PCI function (sysfs), None when unknown."""
    try:
        props = torch.cuda.get_device_properties(device if device is not None else torch.cuda.current_device())
        bus = f"{props.pci_domain_id:04x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
        with open(f"/sys/bus/pci/devices/{bus}/numa_node") as f:
            node = int(f.read().strip())
        return node if node >= 0 else None
    except (OSError, ValueError, AttributeError, RuntimeError):
        return None


def bind_to_gpu_node(device=None) -> tuple[set | None, int | None]:
    """Pin this process's threads to the CPUs of the GPU's NUMA node, so the step's
    launch loop runs next to the GPU and pinned staging buffers are placed on that
    node (first touch).  Returns (previous affinity, node) for ``os.sched_setaffinity``
    to restore; (None, None) when the node or its CPU list is unknown."""
    node = gpu_numa_node(device)
    if node is None or not hasattr(os, "sched_setaffinity"):
        return None, None
    try:
        with open(f"/sys/devices/system/node/node{node}/cpulist") as f:
            spec = f.read().strip()
        cpus = set()
        for part in spec.split(","):
            lo, _, hi = part.partition("-")
            cpus.update(range(int(lo), int(hi or lo) + 1))
        prev = os.sched_getaffinity(0)
        cpus &= prev
        if not cpus:
            return None, None
        os.sched_setaffinity(0, cpus)
        return prev, node
    except (OSError, ValueError):
        return None, None


class HostLatentStore:
    """[pools, rows_per_pool] latent rows of 656 B in page-locked, device-mapped host
    memory, laid out at the ESS_HOST_ROW_PITCH (704-B) pitch so every row starts on a
    64-B host-link request boundary.  ``host`` is the [pools, rows, 656] view."""

    def __init__(self, num_pools: int, rows_per_pool: int, hugepages: bool = True,
                 numa_node: int | None = None, device=None, vmm: bool | None = None):
        _lib.require_cuda()
        if vmm is None:
            vmm = HOST_VMM
        self.num_pools, self.rows_per_pool = num_pools, rows_per_pool
        self.row_bytes, self.pitch = LATENT_BLOCK_BYTES, _lib.HOST_ROW_PITCH
        n = num_pools * rows_per_pool * self.pitch
        node = gpu_numa_node(device) if numa_node is None else numa_node
        hp, alias, placed = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_int32(0)
        flags = (_lib.ESS_HOST_HUGEPAGES if hugepages else 0) | (_lib.ESS_HOST_VMM if vmm else 0)
        _lib.check(_lib.load().ess_host_alloc(n, flags,
                                              -1 if node is None else node, ctypes.byref(hp),
                                              ctypes.byref(alias), ctypes.byref(placed)),
                   "ess_host_alloc")
        self._host_ptr, self._nbytes = hp.value, n
        self.hugepages = bool(placed.value & _lib.ESS_HOST_HUGEPAGES)
        self.vmm = bool(placed.value & _lib.ESS_HOST_VMM)
        self.numa_node = node if placed.value & _lib.ESS_HOST_NUMA_BOUND else None
        raw = (ctypes.c_uint8 * n).from_address(hp.value)
        self._buf = torch.frombuffer(raw, dtype=torch.uint8).view(num_pools, rows_per_pool, self.pitch)
        self.host = self._buf[:, :, :self.row_bytes]
        self.device_ptr = alias.value
        self._registered = True

    @property
    def nbytes(self) -> int:
        return self._nbytes

    def pool_ptr(self, begin: int) -> int:
        return self.device_ptr + begin * self.rows_per_pool * self.pitch

    def close(self):
        if getattr(self, "_registered", False):
            torch.cuda.synchronize()
            self._registered = False
            self.host = self._buf = None
            _lib.load().ess_host_free(self._host_ptr, self._nbytes)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def gather(pool: PoolSet, store: HostLatentStore, acc: AccessBatch, begin: int = 0,
           store_begin: int | None = None, max_ctas: int = 32, exclusive: bool = False,
           stream=None, landed: torch.Tensor | None = None, bulk: bool | None = None,
           pdl: bool = False) -> None:
    """Copy every miss row host[pool][miss_id] -> slot store[pool][miss_row] (K4),
    dequantising to the slot format on the way.  ``exclusive`` keeps the gather off
    SMs that run attention CTAs (overlapped schedule).  ``landed`` (int32 [num],
    zero before the step; sparse_mla_da re-zeroes it) counts each request's landed rows.
    ``pdl``: launched programmatically behind the split on the same stream (ESS_LAUNCH_PDL)."""
    num = acc.counts.shape[0]
    sb = begin if store_begin is None else store_begin
    flags = _lib.ESS_GATHER_EXCLUSIVE_SM if exclusive else 0
    if GATHER_BULK if bulk is None else bulk:
        flags |= _lib.ESS_GATHER_BULK
    if pdl:
        flags |= _lib.ESS_LAUNCH_PDL
    if landed is not None and (landed.dtype != torch.int32 or landed.numel() < num):
        raise ValueError("landed must be int32 with one counter per request")
    _lib.check(_lib.load().ess_gather_signal(
        pool.handle, begin, num, store.pool_ptr(sb), store.rows_per_pool,
        acc.miss_ids.data_ptr(), acc.miss_row.data_ptr(), acc.counts.data_ptr(),
        acc.miss_ids.stride(0), _lib.ptr(landed), max_ctas, flags, _lib.stream_handle(stream)),
        "ess_gather")


def gather_stream(pool: PoolSet, store: HostLatentStore, acc: AccessBatch, ready: torch.Tensor,
                  claim: torch.Tensor, landed: torch.Tensor | None, begin: int = 0, max_ctas: int = 20,
                  exclusive: bool = True, stream=None) -> None:
    """K4 of the streamed step (ess_gather_stream): launched with the step, it fetches each
    request's misses once ``ready`` (ess_topk_split_stream) publishes its split; ``claim``
    (int32 [num], zero at launch) hands out chunks of each miss list to the warps."""
    num = acc.counts.shape[0]
    for t, name in ((ready, "ready"), (claim, "claim")):
        if t.dtype != torch.int32 or t.numel() < num:
            raise ValueError(f"{name} must be int32 with one entry per request")
    flags = _lib.ESS_GATHER_EXCLUSIVE_SM if exclusive else 0
    _lib.check(_lib.load().ess_gather_stream(
        pool.handle, begin, num, store.pool_ptr(begin), store.rows_per_pool,
        acc.miss_ids.data_ptr(), acc.miss_row.data_ptr(), acc.counts.data_ptr(), acc.miss_ids.stride(0),
        ready.data_ptr(), claim.data_ptr(), _lib.ptr(landed), max_ctas, flags, _lib.stream_handle(stream)),
        "ess_gather_stream")


def write_generated(pool: PoolSet, store: HostLatentStore, ids: torch.Tensor, m: torch.Tensor,
                    slots: torch.Tensor, rows: torch.Tensor, begin: int = 0,
                    store_begin: int | None = None, stream=None) -> None:
    """New rows [num, M, 656] -> host store (D2H) and their pool slots."""
    num = ids.shape[0]
    sb = begin if store_begin is None else store_begin
    _lib.check(_lib.load().ess_write_generated(
        pool.handle, begin, num, ids.data_ptr(), m.data_ptr(), slots.data_ptr(), ids.stride(0),
        rows.data_ptr(), store.pool_ptr(sb), store.rows_per_pool, _lib.stream_handle(stream)),
        "ess_write_generated")
