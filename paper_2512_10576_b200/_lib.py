"""ctypes binding of libess_b200.so (include/ess_b200.h).

The product path has exactly one implementation: the sm_100a kernels behind this
library.  If the library is missing or no CUDA device is present, calls fail
loudly — there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# ESS_LIB overrides the library path (scratch variant builds for A/B timing)
LIB_PATH = os.environ.get("ESS_LIB") or os.path.join(_HERE, "libess_b200.so")

V, I32, I64, F32, SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_size_t
PI32, PI64, PV = ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_void_p)

# name -> argtypes (restype int unless noted); mirrors include/ess_b200.h
SIGNATURES = {
    "ess_version": ([], ctypes.c_char_p),
    "ess_status_string": ([ctypes.c_int], ctypes.c_char_p),
    "ess_preload": ([], ctypes.c_int),
    "ess_host_row_pitch": ([], ctypes.c_int),
    "ess_host_register": ([V, SZ, PV], ctypes.c_int),
    "ess_host_unregister": ([V], ctypes.c_int),
    "ess_timestamp": ([V, V], ctypes.c_int),
    "ess_copy_many": ([I32, PV, PV, PI64, V], ctypes.c_int),
    "ess_host_alloc": ([SZ, I32, I32, PV, PV, PI32], ctypes.c_int),
    "ess_host_free": ([V, SZ], ctypes.c_int),
    "ess_pool_create": ([PV, I32, I64, I32, I32, I32], ctypes.c_int),
    "ess_pool_destroy": ([V], ctypes.c_int),
    "ess_pool_reset": ([V, I32, I32, V, V], ctypes.c_int),
    "ess_pool_grow": ([V, I32, I32, V, V], ctypes.c_int),
    "ess_pool_warmup": ([V, I32, I32, V, V, I32, V, V], ctypes.c_int),
    "ess_pool_access": ([V, I32, I32, V, V, I32, V, V, V, V, V, V, V, I32, I32, V], ctypes.c_int),
    "ess_pool_access_mtp": ([V, I32, I32, I32, V, V, I32, V, V, V, V, V, V, V, I32, V, V, V, V, I32, V],
                            ctypes.c_int),
    "ess_pool_append": ([V, I32, I32, V, V, I32, V, V], ctypes.c_int),
    "ess_pool_split": ([V, I32, I32, V, V, I32, V, V, V, V, I32, V], ctypes.c_int),
    "ess_pool_settle": ([V, I32, I32, V, V, I32, V], ctypes.c_int),
    "ess_pool_admit": ([V, I32, I32, V, V, ctypes.c_double, V, I32, V, I64, V, V], ctypes.c_int),
    "ess_pool_lru_order": ([V, I32, I32, V, V, V], ctypes.c_int),
    "ess_pool_counters": ([V, I32, I32, V, V], ctypes.c_int),
    "ess_pool_lookup": ([V, I32, V, I32, V, V], ctypes.c_int),
    "ess_pool_copy_state": ([V, I32, V, I32, I32, V], ctypes.c_int),
    "ess_pool_status": ([V, PI32], ctypes.c_int),
    "ess_pool_info": ([V, PI32, PI64, PI32, PI32, PI64, PV], ctypes.c_int),
    "ess_gather": ([V, I32, I32, V, I64, V, V, V, I32, I32, I32, V], ctypes.c_int),
    "ess_gather_signal": ([V, I32, I32, V, I64, V, V, V, I32, V, I32, I32, V], ctypes.c_int),
    "ess_write_generated": ([V, I32, I32, V, V, V, I32, V, V, I64, V], ctypes.c_int),
    "ess_indexer_logits": ([V, V, V, V, V, I32, I64, V, V], ctypes.c_int),
    "ess_indexer_logits_ex": ([V, V, V, V, V, I32, I64, V, I32, V], ctypes.c_int),
    "ess_indexer_logits_mtp": ([V, V, V, V, V, I32, I32, I64, V, I32, V], ctypes.c_int),
    "ess_indexer_logits_stream": ([V, V, V, V, V, I32, I64, V, I32, I32, V, V], ctypes.c_int),
    "ess_topk_split_stream": ([V, I64, V, I32, I32, V, I32, V, V, I32, V, V, V, V, I32, V, V, I32, V],
                              ctypes.c_int),
    "ess_gather_stream": ([V, I32, I32, V, I64, V, V, V, I32, V, V, V, I32, I32, V], ctypes.c_int),
    "ess_topk": ([V, I64, V, I32, I32, V, I32, V, V], ctypes.c_int),
    "ess_topk_mtp": ([V, I64, V, I32, I32, I32, V, I32, V, V], ctypes.c_int),
    "ess_topk_split": ([V, I64, V, I32, I32, V, I32, V, V, I32, V, V, V, V, I32, V], ctypes.c_int),
    "ess_topk_split_ex": ([V, I64, V, I32, I32, V, I32, V, V, I32, V, V, V, V, I32, I32, V], ctypes.c_int),
    "ess_sparse_mla": ([V, I32, V, V, I32, V, I32, I32, F32, V, V, V, V, I32, V], ctypes.c_int),
    "ess_sparse_mla_da": ([V, I32, V, V, V, I32, V, I32, V, I32, F32, V, V, V], ctypes.c_int),
    "ess_sparse_mla_da_split": ([V, I32, V, V, V, I32, V, I32, V, I32, F32, V, V, V, V, I32, V],
                                ctypes.c_int),
}

ESS_OK = 0
ESS_ERR_CAPACITY, ESS_ERR_SHRINK, ESS_ERR_DUPLICATE = -1, -2, -3
ESS_ERR_NOMEM, ESS_ERR_RATIO, ESS_ERR_ARG, ESS_ERR_CUDA, ESS_ERR_CLOCK = -4, -5, -6, -7, -8
ESS_ERR_RANGE = -9
ESS_ACCESS_SORT_EVICTED = 1
ESS_MLA_PARTIAL, ESS_MLA_RESUME = 1, 2
ESS_MLA_SPLIT_SHIFT, ESS_MLA_MAX_SPLIT = 8, 8
ESS_MLA_QTOK_SHIFT = 12
MAX_QTOK = 4  # ESS_INDEXER_MAX_QTOK: query tokens per request and step (MTP width + 1)
ESS_GATHER_EXCLUSIVE_SM = 1
ESS_GATHER_BULK = 2
ESS_LAUNCH_PDL = 1 << 30
ESS_HOST_HUGEPAGES, ESS_HOST_NUMA_BOUND, ESS_HOST_VMM = 1, 2, 4
MAX_REQUEST = 2048
LATENT_ROW_BYTES = 656   # host store / transfer format (e4m3 NoPE + scales + bf16 RoPE)
# host store row pitch (64-B aligned rows; ESS_HOST_ROW_PITCH); the env override pairs with
# a scratch library built with the same -DESS_HOST_ROW_PITCH
HOST_ROW_PITCH = int(os.environ.get("ESS_HOST_ROW_PITCH", "704"))
# GPU slot store formats (include/ess_b200.h): the raw 656-B latent row, dequantised in
# shared memory by the CTA-pair FP8 K5 (mla2.cu), or 576 x f16 dequantised on admission
# (mla.cu).  ESS_SLOT_FORMAT picks the decode layer's default.
SLOT_ROW_BYTES_FP8, SLOT_ROW_BYTES_F16 = 656, 1152
SLOT_FORMATS = {"fp8": SLOT_ROW_BYTES_FP8, "f16": SLOT_ROW_BYTES_F16}
SLOT_ROW_BYTES = SLOT_FORMATS[os.environ.get("ESS_SLOT_FORMAT", "f16")]

_lib = None


def load():
    """Load the library (no CUDA calls).  Raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing; build it with "
                              "`python -m paper_2512_10576_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        if L.ess_host_row_pitch() != HOST_ROW_PITCH:
            raise ImportError(f"{LIB_PATH} was built with host row pitch {L.ess_host_row_pitch()}, "
                              f"the Python side uses {HOST_ROW_PITCH} (ESS_HOST_ROW_PITCH)")
        _lib = L
    return _lib


def status_text(rc: int) -> str:
    return load().ess_status_string(rc).decode()


def check(rc: int, what: str = "") -> None:
    """Map an ESS_* status to the reference's exception classes."""
    if rc == ESS_OK:
        return
    msg = f"{what}: {status_text(rc)}" if what else status_text(rc)
    if rc in (ESS_ERR_CAPACITY, ESS_ERR_SHRINK, ESS_ERR_DUPLICATE, ESS_ERR_RATIO, ESS_ERR_ARG, ESS_ERR_RANGE):
        raise ValueError(msg)
    if rc == ESS_ERR_NOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None passes NULL)."""
    return None if t is None else t.data_ptr()


def stream_handle(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


_PRELOADED = set()


def require_cuda(t=None) -> None:
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("ess_b200 needs a CUDA device (sm_100a); no CPU fallback exists")
    if t is not None and not t.is_cuda:
        raise ValueError("tensor must be on the CUDA device")
    dev = torch.cuda.current_device()
    if dev not in _PRELOADED:
        # every kernel loaded before the first launch: with lazy module loading a kernel's
        # first launch waits for the device, which deadlocks the streamed hand-offs
        check(load().ess_preload(), "ess_preload")
        _PRELOADED.add(dev)


def check_tensor(t, name: str, dtypes, shape=None, contiguous: bool = True, device=None) -> None:
    """Argument validation of the ctypes wrappers: the kernels address tensors through
    raw pointers and the strides they are given, so a wrong dtype, shape or layout must
    be refused here (ValueError), never reach the device."""
    import torch
    if not isinstance(t, torch.Tensor):
        raise ValueError(f"{name} must be a torch.Tensor")
    if not isinstance(dtypes, (tuple, list)):
        dtypes = (dtypes,)
    if t.dtype not in dtypes:
        raise ValueError(f"{name} has dtype {t.dtype}, expected one of {list(dtypes)}")
    if shape is not None:
        if len(shape) != t.dim() or any(w is not None and w != g for w, g in zip(shape, t.shape)):
            raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
    if contiguous and not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if not t.is_cuda or (device is not None and t.device != device):
        raise ValueError(f"{name} must be on the CUDA device {device or ''}".rstrip())


COPY_MAX = 64  # ESS_COPY_MAX


def copy_many(pairs, stream=None) -> None:
    """Device-to-device copies [(dst, src), ...] of contiguous CUDA tensors with equal byte
    sizes, in one SM kernel per 64 pairs (ess_copy_many) — the decode step's input
    staging.  Pairs that are not 16-B aligned / sized take torch's copy."""
    fast = []
    for dst, src in pairs:
        nb = dst.numel() * dst.element_size()
        if (src.dtype != dst.dtype or src.numel() != dst.numel() or not (dst.is_contiguous() and src.is_contiguous())
                or not (dst.is_cuda and src.is_cuda)):
            raise ValueError("copy_many: contiguous CUDA tensors of one dtype and size")
        if nb % 16 or dst.data_ptr() % 16 or src.data_ptr() % 16:
            dst.copy_(src.view(dst.shape), non_blocking=True)
        elif nb:
            fast.append((dst.data_ptr(), src.data_ptr(), nb))
    for i in range(0, len(fast), COPY_MAX):
        chunk = fast[i:i + COPY_MAX]
        n = len(chunk)
        d = (ctypes.c_void_p * n)(*[c[0] for c in chunk])
        sp = (ctypes.c_void_p * n)(*[c[1] for c in chunk])
        b = (ctypes.c_int64 * n)(*[c[2] for c in chunk])
        check(load().ess_copy_many(n, d, sp, b, stream_handle(stream)), "ess_copy_many")
