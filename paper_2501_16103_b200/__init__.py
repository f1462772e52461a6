"""Thin Python binding over libmoe_sm100.so (C ABI in include/moe_sm100.h).

Argument marshalling only: every step of the path (routing buckets, the
compressed mapping decode, the gathered tcgen05 GEMM) runs in the library's
CUDA kernels; the host planner runs in the library's C++ code.  PyTorch is used
for device memory and streams.  There is no CPU fallback: if the library is
missing or the device is not sm_100, calls raise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# MOE_LIB: load another build of the same C ABI (same-box A/B timing of kernel revisions).
LIB_PATH = os.environ.get("MOE_LIB") or os.path.join(HERE, "libmoe_sm100.so")

MOE_OK, MOE_OK_EMPTY = 0, 1
MOE_ERR = {-1: "INVALID", -2: "UNSUPPORTED", -3: "CAPACITY", -4: "CUDA", -5: "NCCL"}
MOE_DTYPE_BF16, MOE_DTYPE_F32, MOE_DTYPE_E4M3 = 0, 1, 2
MOE_EP_UNFUSED = 1
MOE_PAD_MAX, MOE_PAD_REPEAT, MOE_SPLIT_TAIL = 0, 1, 2
MOE_ORDER_ALTERNATING, MOE_ORDER_HALF_INTERVAL, MOE_ORDER_LIGHT_LAST = 4, 8, 4096
MOE_LIGHT_ROWS = 64
MOE_GRID_BALANCED, MOE_GRID_STATIC, MOE_A_GATHER4, MOE_EPI_REGISTER, MOE_SCHED_DYNAMIC = 16, 32, 64, 128, 256
MOE_L2_PREFETCH = 512
MOE_SPLIT_K = 1024
MOE_SCHED_HALF_LAST = 2048
MOE_SCHED_PLAN_ORDER = 16384
MOE_ROUTE_NO_SMALL, MOE_ROUTE_THREE_KERNELS = 1, 2
MOE_KIND_WIDE, MOE_KIND_SWAP, MOE_MAX_RULES = 0, 1, 2
MOE_DEFAULT_SWAP_MAX = 64                       # include/moe_sm100.h: the swap-AB rule of tests and A/B runs
MOE_KIND_GEMV, MOE_DEFAULT_GEMV_MAX, MOE_GEMV_MIN_TILES = 2, 4, 128
MOE_KIND_RIDE, MOE_RIDE_MAX_ROWS = 3, 32
DEFAULT_CATALOG = ((MOE_KIND_GEMV, MOE_DEFAULT_GEMV_MAX),)   # the built-in catalog of wide pair plans


class _Rule(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("m_max", ctypes.c_int32)]


def parse_catalog(text: str):
    """'kind.m_max+kind.m_max' (e.g. '2.4+1.64'), 'none' (one strategy) or 'default' -> a catalog argument."""
    text = text.strip()
    if text in ("", "default"):
        return None
    if text == "none":
        return ()
    rules = tuple(tuple(int(x) for x in r.split(".")) for r in text.split("+"))
    if len(rules) > MOE_MAX_RULES or any(len(r) != 2 for r in rules):
        raise ValueError(f"MOE_TILE_CATALOG: at most {MOE_MAX_RULES} 'kind.m_max' rules, got {text!r}")
    return rules


# SURVEY §5 config override: the tile-strategy catalog of plans built without an explicit one, read once at
# import (the library itself reads no environment; the catalog reaches it as plan arguments).
ENV_CATALOG = parse_catalog(os.environ.get("MOE_TILE_CATALOG", ""))


def _rules(catalog):
    """None -> MOE_TILE_CATALOG if set, else the built-in catalog (n_rules = -1); a sequence of (kind, m_max)
    -> the rule array."""
    if catalog is None:
        catalog = ENV_CATALOG
    if catalog is None:
        return None, -1
    arr = (_Rule * max(len(catalog), 1))(*[_Rule(int(k), int(m)) for k, m in catalog])
    return arr, len(catalog)
MOE_PLAN_MAGIC = 0x4D4F4531
MOE_PLAN_HEADER = 16
MOE_PLAN_TASK_WORDS = 8

# Public symbols of include/moe_sm100.h, moe_sm100_ep.h, moe_sm100_ffn.h, moe_sm100_fp8.h and moe_sm100_debug.h.
EXPORTED = (
    "moe_plan_blob_words", "moe_plan_build", "moe_plan_create", "moe_plan_update", "moe_plan_query",
    "moe_plan_blob", "moe_plan_device_blob", "moe_plan_destroy", "moe_route", "moe_gemm",
    "moe_decode_debug", "moe_device_info", "moe_last_error", "moe_version", "moe_probe_gather4",
    "moe_gemm_profile", "moe_plan_device", "moe_plan_sync", "moe_gemm_rowmap",
    "moe_ep_dispatch_plan", "moe_gather_rows", "moe_ep_combine_map", "moe_ep_unpack", "moe_route_plan",
    "moe_gemm_swiglu", "moe_combine", "moe_gemm_fp8", "moe_gemm_fp8_rowmap", "moe_gemm_fp8_profile",
    "moe_ep_unique_id", "moe_ep_create", "moe_ep_forward", "moe_ep_last_rows", "moe_ep_last_gemm_ms",
    "moe_ep_destroy", "moe_ep_create_loopback", "moe_ep_combine_ptr", "moe_gemm_rowptr",
    "moe_route_ex", "moe_plan_suggest_tile", "moe_plan_create_expected", "moe_plan_build_catalog",
    "moe_plan_create_catalog", "moe_ep_peer_create", "moe_ep_peer_connect", "moe_ep_peer_output",
    "moe_ep_peer_set_timeout", "moe_ep_peer_status",
)


class MoeError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"moe status {status} ({MOE_ERR.get(status, '?')}): {msg}")
        self.status = status


_lib = None


def lib() -> ctypes.CDLL:
    """Load the in-tree library (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} missing: run `python -m paper_2501_16103_b200.build` "
                           "(or __graft_entry__.build()) — there is no fallback path")
    L = ctypes.CDLL(LIB_PATH)
    c_i32p = ctypes.POINTER(ctypes.c_int32)
    c_i64p = ctypes.POINTER(ctypes.c_int64)
    vp = ctypes.c_void_p
    sig = {
        "moe_plan_blob_words": (ctypes.c_int64, [ctypes.c_int32]),
        "moe_plan_build": (ctypes.c_int32, [c_i32p, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                            ctypes.c_int32, ctypes.c_uint32, c_i32p, ctypes.c_int64, c_i64p]),
        "moe_plan_create": (ctypes.c_int32, [c_i32p, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                             ctypes.c_int32, ctypes.c_uint32, vp, ctypes.POINTER(vp)]),
        "moe_plan_build_catalog": (ctypes.c_int32, [c_i32p, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64,
                                                    ctypes.c_int32, ctypes.c_int32, ctypes.c_uint32, vp, ctypes.c_int32,
                                                    c_i32p, ctypes.c_int64, c_i64p]),
        "moe_plan_create_catalog": (ctypes.c_int32, [c_i32p, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64,
                                                     ctypes.c_int32, ctypes.c_int32, ctypes.c_uint32, vp,
                                                     ctypes.c_int32, vp, ctypes.POINTER(vp)]),
        "moe_plan_update": (ctypes.c_int32, [vp, c_i32p, vp]),
        "moe_plan_query": (ctypes.c_int32, [vp, c_i32p, c_i32p, c_i32p]),
        "moe_plan_blob": (ctypes.c_int32, [vp, c_i32p, ctypes.c_int64, c_i64p]),
        "moe_plan_device_blob": (vp, [vp]),
        "moe_plan_destroy": (None, [vp]),
        "moe_route": (ctypes.c_int32, [vp, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, vp, vp, vp, vp, vp, vp]),
        "moe_route_plan": (ctypes.c_int32, [vp, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, vp, vp, vp, vp, vp,
                                            vp, vp]),
        "moe_route_ex": (ctypes.c_int32, [vp, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, vp, vp, vp, vp, vp,
                                          vp, ctypes.c_uint32, vp]),
        "moe_plan_suggest_tile": (ctypes.c_int32, [ctypes.c_int64, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64,
                                                   c_i32p, c_i32p]),
        "moe_plan_create_expected": (ctypes.c_int32, [ctypes.c_int64, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64,
                                                      ctypes.c_int32, ctypes.c_int32, ctypes.c_uint32, vp,
                                                      ctypes.POINTER(vp)]),
        "moe_gemm": (ctypes.c_int32, [vp, vp, ctypes.c_int64, vp, vp, vp, ctypes.c_int32, vp]),
        "moe_decode_debug": (ctypes.c_int32, [vp, vp, vp]),
        "moe_device_info": (ctypes.c_int32, [c_i32p, c_i32p, c_i32p]),
        "moe_last_error": (ctypes.c_char_p, []),
        "moe_version": (ctypes.c_char_p, []),
        "moe_probe_gather4": (ctypes.c_int32, [vp, ctypes.c_int64, ctypes.c_int64, vp, ctypes.c_int32, vp, vp]),
        "moe_gemm_profile": (ctypes.c_int32, [vp, vp, ctypes.c_int64, vp, vp, vp, ctypes.c_int32, vp, vp]),
        "moe_plan_device": (ctypes.c_int32, [vp, vp, vp]),
        "moe_plan_sync": (ctypes.c_int32, [vp, vp]),
        "moe_gemm_rowmap": (ctypes.c_int32, [vp, vp, ctypes.c_int64, vp, vp, vp, ctypes.c_int32, vp, vp]),
        "moe_ep_dispatch_plan": (ctypes.c_int32, [vp, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                                  ctypes.c_int32, vp, vp, vp, vp, vp]),
        "moe_gather_rows": (ctypes.c_int32, [vp, vp, ctypes.c_int64, ctypes.c_int64, vp, vp]),
        "moe_ep_combine_map": (ctypes.c_int32, [vp, vp, ctypes.c_int64, vp, vp, ctypes.c_int32, ctypes.c_int32,
                                                vp, vp, vp, vp]),
        "moe_ep_unpack": (ctypes.c_int32, [vp, vp, ctypes.c_int64, vp, vp, vp, ctypes.c_int32, ctypes.c_int32,
                                           ctypes.c_int64, vp, vp]),
        "moe_gemm_swiglu": (ctypes.c_int32, [vp, vp, ctypes.c_int64, vp, vp, vp, vp, ctypes.c_int32, vp]),
        "moe_gemm_fp8": (ctypes.c_int32, [vp, vp, ctypes.c_int64, vp, vp, vp, vp, ctypes.c_int32, vp]),
        "moe_gemm_fp8_rowmap": (ctypes.c_int32, [vp, vp, ctypes.c_int64, vp, vp, vp, vp, ctypes.c_int32, vp, vp]),
        "moe_gemm_fp8_profile": (ctypes.c_int32, [vp, vp, ctypes.c_int64, vp, vp, vp, vp, ctypes.c_int32, vp, vp]),
        "moe_ep_unique_id": (ctypes.c_int32, [vp]),
        "moe_ep_create": (ctypes.c_int32, [vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                           ctypes.c_int32, ctypes.c_uint32, ctypes.POINTER(vp)]),
        "moe_ep_forward": (ctypes.c_int32, [vp, vp, ctypes.c_int64, ctypes.c_int32, vp, ctypes.c_int64,
                                            ctypes.c_int32, vp, ctypes.c_int64, vp, vp, ctypes.c_int32, vp]),
        "moe_ep_last_rows": (ctypes.c_int32, [vp, c_i64p, c_i64p, c_i64p]),
        "moe_ep_last_gemm_ms": (ctypes.c_int32, [vp, ctypes.POINTER(ctypes.c_float)]),
        "moe_ep_create_loopback": (ctypes.c_int32, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                                    ctypes.c_int32, ctypes.POINTER(vp)]),
        "moe_ep_combine_ptr": (ctypes.c_int32, [vp, vp, ctypes.c_int64, vp, ctypes.c_int32, ctypes.c_int32, vp, vp, vp,
                                                vp, ctypes.c_int64, vp, vp]),
        "moe_gemm_rowptr": (ctypes.c_int32, [vp, vp, ctypes.c_int64, vp, vp, ctypes.c_int32, vp, vp, ctypes.c_int32,
                                             vp]),
        "moe_ep_destroy": (None, [vp]),
        "moe_ep_peer_create": (ctypes.c_int32, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                                ctypes.c_int32, ctypes.c_int64, ctypes.c_int32, ctypes.c_int64,
                                                ctypes.c_int64, ctypes.POINTER(vp), vp]),
        "moe_ep_peer_connect": (ctypes.c_int32, [vp, vp]),
        "moe_ep_peer_output": (ctypes.c_int32, [vp, ctypes.POINTER(vp), c_i64p]),
        "moe_ep_peer_set_timeout": (ctypes.c_int32, [vp, ctypes.c_int64]),
        "moe_ep_peer_status": (ctypes.c_int32, [vp, c_i32p]),
        "moe_combine": (ctypes.c_int32, [vp, ctypes.c_int32, ctypes.c_int64, ctypes.c_int32, ctypes.c_int64, vp, vp,
                                         vp, ctypes.c_int32, vp, vp, ctypes.c_int32, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _check(status: int) -> int:
    if status < 0:
        raise MoeError(status, lib().moe_last_error().decode())
    return status


def _i32ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


# ---------------------------------------------------------------------------
# plan (host, no GPU needed)
# ---------------------------------------------------------------------------
def moe_plan_build(counts, H: int, N: int, bm: int = 0, bn: int = 0, flags: int = MOE_PAD_MAX,
                   catalog=None) -> np.ndarray:
    """The compressed mapping blob (int32 words, layout in include/moe_sm100.h).
    catalog: None = the built-in tile-strategy catalog, () = one strategy, else (kind, m_max) rules."""
    c = np.ascontiguousarray(np.asarray(counts, dtype=np.int32))
    E = int(c.shape[0])
    L = lib()
    cap = int(L.moe_plan_blob_words(E)) if E > 0 else 64
    blob = np.zeros(max(cap, 16), dtype=np.int32)
    n = ctypes.c_int64(0)
    rules, nr = _rules(catalog)
    _check(L.moe_plan_build_catalog(_i32ptr(c), E, H, N, bm, bn, flags, rules, nr, _i32ptr(blob), blob.size,
                                    ctypes.byref(n)))
    return blob[: n.value].copy()


def parse_plan_blob(blob: np.ndarray) -> dict:
    """Split a blob into named arrays (layout of include/moe_sm100.h)."""
    b = np.asarray(blob)
    if int(b[0]) != MOE_PLAN_MAGIC:
        raise ValueError("not a plan blob")
    M, total, M_pad, E, N, H, bm, bn, n_tasks, flags = (int(x) for x in b[1:11])
    catalog = tuple((int(b[12 + 2 * i]), int(b[13 + 2 * i])) for i in range(MOE_MAX_RULES) if b[13 + 2 * i] >= 0)
    o = MOE_PLAN_HEADER
    prefix = b[o:o + M_pad]
    sigma = b[o + M_pad:o + 2 * M_pad]
    po = o + 2 * M_pad
    params = b[po:po + MOE_PLAN_TASK_WORDS * n_tasks].reshape(n_tasks, MOE_PLAN_TASK_WORDS)
    row_off = b[po + MOE_PLAN_TASK_WORDS * n_tasks: po + MOE_PLAN_TASK_WORDS * n_tasks + E + 1]
    return dict(M=M, total=total, M_pad=M_pad, E=E, N=N, H=H, bm=bm, bn=bn, n_tasks=n_tasks, flags=flags,
                prefix=prefix, sigma=sigma, params=params, row_off=row_off, catalog=catalog)


def _stream(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def suggest_tile(rows: int, E: int, H: int, N: int) -> tuple[int, int]:
    """Tile shape (bm, bn) the library's automatic rule picks for `rows` routed rows spread evenly over
    min(E, rows) experts (moe_plan_suggest_tile) — for plans created before the counts exist."""
    bm, bn = ctypes.c_int32(), ctypes.c_int32()
    _check(lib().moe_plan_suggest_tile(int(rows), int(E), int(H), int(N), ctypes.byref(bm), ctypes.byref(bn)))
    return bm.value, bn.value


class Plan:
    """Device-resident plan (moe_plan_create / moe_plan_update / moe_plan_destroy)."""

    def __init__(self, counts, H: int, N: int, bm: int = 0, bn: int = 0, flags: int = MOE_PAD_MAX,
                 stream=None, E: int | None = None, catalog=None):
        """counts: host int array [E], or None (with E=...) for a plan filled by update_device().
        catalog: None = the built-in tile-strategy catalog, () = one strategy, else (kind, m_max) rules."""
        if counts is None:
            c, cp = None, None
            self.E = int(E)
        else:
            c = np.ascontiguousarray(np.asarray(counts, dtype=np.int32))
            cp = _i32ptr(c)
            self.E = int(c.shape[0])
        self.H, self.N, self.bn, self.flags = H, N, bn, flags
        self._h = ctypes.c_void_p()
        rules, nr = _rules(catalog)
        self.status = _check(lib().moe_plan_create_catalog(cp, self.E, H, N, bm, bn, flags, rules, nr,
                                                           _stream(stream), ctypes.byref(self._h)))
        b = self.blob()
        self.bm, self.bn = int(b[7]), int(b[8])  # resolved tile shape (0: automatic)
        self.catalog = parse_plan_blob(b)["catalog"]
        self.device_resident = False

    def update_device(self, counts_dev, stream=None):
        """Re-plan on the device from device counts (no host synchronisation)."""
        _check(lib().moe_plan_device(self._h, counts_dev.data_ptr(), _stream(stream)))
        self.device_resident = True

    def sync(self, stream=None) -> int:
        """Copy a device-built plan back to the host (synchronises the stream)."""
        self.status = _check(lib().moe_plan_sync(self._h, _stream(stream)))
        self.device_resident = False
        return self.status

    def update(self, counts, stream=None) -> int:
        c = np.ascontiguousarray(np.asarray(counts, dtype=np.int32))
        self.status = _check(lib().moe_plan_update(self._h, _i32ptr(c), _stream(stream)))
        self.device_resident = False
        return self.status

    def query(self) -> tuple[int, int, int]:
        M, total, M_pad = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        _check(lib().moe_plan_query(self._h, ctypes.byref(M), ctypes.byref(total), ctypes.byref(M_pad)))
        return M.value, total.value, M_pad.value

    @property
    def total_tiles(self) -> int:
        return self.query()[1]

    def blob(self) -> np.ndarray:
        n = ctypes.c_int64()
        _check(lib().moe_plan_blob(self._h, None, 0, ctypes.byref(n)))
        out = np.zeros(n.value, dtype=np.int32)
        _check(lib().moe_plan_blob(self._h, _i32ptr(out), out.size, ctypes.byref(n)))
        return out

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            lib().moe_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# device entry points
# ---------------------------------------------------------------------------
def moe_device_info() -> tuple[int, int, int]:
    n, ma, mi = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    _check(lib().moe_device_info(ctypes.byref(n), ctypes.byref(ma), ctypes.byref(mi)))
    return n.value, ma.value, mi.value


def moe_route(topk_ids, E: int, with_slot: bool = True, stream=None, plan: "Plan | None" = None,
              route_flags: int = 0):
    """topk_ids: int32 CUDA tensor [T, k] -> (counts[E], row_off[E+1], token_idx[T*k], slot, status).

    With masked (negative) or invalid ids only the first sum(counts) = row_off[E] entries of
    token_idx / slot are meaningful (the length is not read back, to avoid a host sync)."""
    import torch

    assert topk_ids.is_cuda and topk_ids.dtype == torch.int32 and topk_ids.is_contiguous()
    T, k = topk_ids.shape
    dev = topk_ids.device
    counts = torch.empty(E, dtype=torch.int32, device=dev)
    row_off = torch.empty(E + 1, dtype=torch.int32, device=dev)
    token_idx = torch.empty(max(T * k, 1), dtype=torch.int32, device=dev)
    slot = torch.empty(max(T * k, 1), dtype=torch.int32, device=dev) if with_slot else None
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    args = (topk_ids.data_ptr(), T, k, E, counts.data_ptr(), row_off.data_ptr(), token_idx.data_ptr(),
            slot.data_ptr() if slot is not None else None, status.data_ptr())
    if route_flags:                              # explicit kernel path (moe_route_ex)
        _check(lib().moe_route_ex(*args, plan.handle if plan is not None else None, route_flags, _stream(stream)))
    elif plan is None:
        _check(lib().moe_route(*args, _stream(stream)))
    else:                                        # fused with the device planner (moe_route_plan)
        _check(lib().moe_route_plan(*args, plan.handle, _stream(stream)))
    if plan is not None:
        plan.device_resident = True
    return counts, row_off, token_idx[: T * k], (slot[: T * k] if slot is not None else None), status


def moe_gemm(plan: Plan, X, token_idx, W, Y=None, out_dtype=None, stream=None, row_map=None):
    """Y[sum m_e, N] = per-expert X[token_idx] @ W[e] in one launch (row_map: Y row of CSR row i).
    token_idx None: X's rows are already in CSR order (X row i = CSR row i)."""
    import torch

    out_dtype = out_dtype or torch.bfloat16
    assert X.is_cuda and X.dtype == torch.bfloat16 and X.is_contiguous()
    assert W.is_cuda and W.dtype == torch.bfloat16 and W.is_contiguous()
    if token_idx is not None:
        assert token_idx.dtype == torch.int32 and token_idx.is_contiguous()
    rows = int(token_idx.numel()) if token_idx is not None else int(X.shape[0])
    tp = token_idx.data_ptr() if token_idx is not None else None
    if Y is None:
        Y = torch.empty((rows, plan.N), dtype=out_dtype, device=X.device)
    yd = MOE_DTYPE_F32 if Y.dtype == torch.float32 else MOE_DTYPE_BF16
    if row_map is None:
        _check(lib().moe_gemm(plan.handle, X.data_ptr(), X.shape[0], tp, W.data_ptr(),
                              Y.data_ptr(), yd, _stream(stream)))
    else:
        assert row_map.dtype == torch.int32 and row_map.is_contiguous()
        _check(lib().moe_gemm_rowmap(plan.handle, X.data_ptr(), X.shape[0], tp, W.data_ptr(),
                                     Y.data_ptr(), yd, row_map.data_ptr(), _stream(stream)))
    return Y


def moe_gemm_fp8(plan: Plan, X, token_idx, W, scale=None, Y=None, out_dtype=None, stream=None, row_map=None):
    """Y[sum m_e, N] = scale[e] * (X[token_idx] @ W[e]) on FP8 E4M3 X [T, H] and W [E, H, N]
    (torch.float8_e4m3fn or uint8 codes), fp32 accumulate, one launch (include/moe_sm100_fp8.h).
    scale: [E] fp32 device tensor or None; token_idx None: X's rows are already in CSR order;
    row_map: Y row of CSR row i (moe_gemm_fp8_rowmap)."""
    import torch

    out_dtype = out_dtype or torch.bfloat16
    f8 = (torch.float8_e4m3fn, torch.uint8)
    assert X.is_cuda and X.dtype in f8 and X.is_contiguous()
    assert W.is_cuda and W.dtype in f8 and W.is_contiguous()
    if token_idx is not None:
        assert token_idx.dtype == torch.int32 and token_idx.is_contiguous()
    if scale is not None:
        assert scale.is_cuda and scale.dtype == torch.float32 and scale.is_contiguous()
    rows = int(token_idx.numel()) if token_idx is not None else int(X.shape[0])
    if Y is None:
        Y = torch.empty((rows, plan.N), dtype=out_dtype, device=X.device)
    yd = MOE_DTYPE_F32 if Y.dtype == torch.float32 else MOE_DTYPE_BF16
    tp = token_idx.data_ptr() if token_idx is not None else None
    sp = scale.data_ptr() if scale is not None else None
    if row_map is None:
        _check(lib().moe_gemm_fp8(plan.handle, X.data_ptr(), X.shape[0], tp, W.data_ptr(), sp, Y.data_ptr(), yd,
                                  _stream(stream)))
    else:
        assert row_map.dtype == torch.int32 and row_map.is_contiguous()
        _check(lib().moe_gemm_fp8_rowmap(plan.handle, X.data_ptr(), X.shape[0], tp, W.data_ptr(), sp, Y.data_ptr(),
                                         yd, row_map.data_ptr(), _stream(stream)))
    return Y


def moe_gemm_swiglu(plan: Plan, X, token_idx, W_gate, W_up, Y=None, out_dtype=None, stream=None):
    """Y[sum m_e, I] = silu(X[token_idx] @ W_gate[e]) * (X[token_idx] @ W_up[e]) in one launch
    (plan: N = I, bm = bn = 256; include/moe_sm100_ffn.h)."""
    import torch

    out_dtype = out_dtype or torch.bfloat16
    for t in (X, W_gate, W_up):
        assert t.is_cuda and t.dtype == torch.bfloat16 and t.is_contiguous()
    assert W_gate.shape == W_up.shape
    assert token_idx.dtype == torch.int32 and token_idx.is_contiguous()
    if Y is None:
        Y = torch.empty((int(token_idx.numel()), plan.N), dtype=out_dtype, device=X.device)
    yd = MOE_DTYPE_F32 if Y.dtype == torch.float32 else MOE_DTYPE_BF16
    _check(lib().moe_gemm_swiglu(plan.handle, X.data_ptr(), X.shape[0], token_idx.data_ptr(), W_gate.data_ptr(),
                                 W_up.data_ptr(), Y.data_ptr(), yd, _stream(stream)))
    return Y


def moe_combine(Y, token_idx, slot, row_off, topk_w, out=None, out_dtype=None, stream=None):
    """out[t] = sum_j topk_w[t, j] * Y[row(t, j)], rows recovered from the route's CSR."""
    import torch

    T, k = int(topk_w.shape[0]), int(topk_w.shape[1])
    N = int(Y.shape[1])
    E = int(row_off.numel()) - 1
    assert topk_w.dtype == torch.float32 and topk_w.is_contiguous() and Y.is_contiguous()
    assert slot is not None and slot.dtype == torch.int32 and token_idx.dtype == torch.int32
    if out is None:
        out = torch.empty((T, N), dtype=out_dtype or torch.bfloat16, device=Y.device)
    yd = MOE_DTYPE_F32 if Y.dtype == torch.float32 else MOE_DTYPE_BF16
    od = MOE_DTYPE_F32 if out.dtype == torch.float32 else MOE_DTYPE_BF16
    _check(lib().moe_combine(Y.data_ptr(), yd, T, k, N, token_idx.data_ptr(), slot.data_ptr(), row_off.data_ptr(), E,
                             topk_w.data_ptr(), out.data_ptr(), od, _stream(stream)))
    return out


class MoeFFN:
    """The full MoE FFN layer on one GPU (R14): route (+ device plan
    for the gated GEMM) -> device plan for the down GEMM -> moe_gemm_swiglu (h in bf16) -> moe_gemm
    (rows in CSR order, no gather; fp32 rows) -> moe_combine.  Every step runs in the library's kernels; nothing
    synchronises with the host, so a step can be captured in one CUDA graph."""

    def __init__(self, W_gate, W_up, W_down, stream=None):
        import torch

        self.E, self.H, self.I = (int(x) for x in W_gate.shape)
        assert W_down.shape == (self.E, self.I, W_down.shape[2])
        self.Ho = int(W_down.shape[2])
        self.Wg, self.Wu, self.Wd = W_gate, W_up, W_down
        self.plan_gu = Plan(None, self.H, self.I, 256, 256, stream=stream, E=self.E)
        self.plan_dn = None
        self._torch = torch

    def forward(self, X, topk_ids, topk_w, out=None, out_dtype=None, stream=None):
        torch = self._torch
        T, k = int(topk_ids.shape[0]), int(topk_ids.shape[1])
        R = T * k
        if self.plan_dn is None:
            bm, bn = suggest_tile(R, self.E, self.I, self.Ho)
            self.plan_dn = Plan(None, self.I, self.Ho, bm, bn, stream=stream, E=self.E)
        counts, row_off, tok, slot, _ = moe_route(topk_ids, self.E, stream=stream, plan=self.plan_gu)
        self.plan_dn.update_device(counts, stream=stream)
        Hmid = moe_gemm_swiglu(self.plan_gu, X, tok, self.Wg, self.Wu, stream=stream)
        # rows already in CSR order; fp32 rows into the combine (no second bf16 rounding, R14)
        Y = moe_gemm(self.plan_dn, Hmid, None, self.Wd, out_dtype=torch.float32, stream=stream)
        out = moe_combine(Y, tok, slot, row_off, topk_w, out=out, out_dtype=out_dtype, stream=stream)
        self.last = dict(counts=counts, row_off=row_off, token_idx=tok, slot=slot, h=Hmid, y=Y)
        return out


PROF_SLOTS = ("mma_wait_tmem", "mma_wait_full", "mma_total", "prod_wait_empty", "epi_wait_full", "epi_work",
              "tiles", "prod_total", "mma_issue", "mma_tile_gap", "b_wait_empty", "b_total", "lat_b", "lat_a",
              "release", "stages")


def moe_gemm_profile(plan: Plan, X, token_idx, W, Y, stream=None, scale=None):
    """Instrumented moe_gemm (FP8 X / W: moe_gemm_fp8_profile): returns Y and per-CTA cycle counters
    [grid, 16] (see moe_sm100_debug.h)."""
    import torch

    n_sm = moe_device_info()[0]
    total = n_sm if plan.device_resident else plan.total_tiles
    grid = min(total, n_sm) if plan.bm == 128 else 2 * min(total, n_sm // 2)
    prof = torch.zeros((max(grid, 1), len(PROF_SLOTS)), dtype=torch.int64, device=X.device)
    yd = MOE_DTYPE_F32 if Y.dtype == torch.float32 else MOE_DTYPE_BF16
    if X.dtype in (torch.uint8, torch.float8_e4m3fn):
        _check(lib().moe_gemm_fp8_profile(plan.handle, X.data_ptr(), X.shape[0], token_idx.data_ptr(), W.data_ptr(),
                                          scale.data_ptr() if scale is not None else None, Y.data_ptr(), yd,
                                          prof.data_ptr(), _stream(stream)))
    else:
        _check(lib().moe_gemm_profile(plan.handle, X.data_ptr(), X.shape[0], token_idx.data_ptr(), W.data_ptr(),
                                      Y.data_ptr(), yd, prof.data_ptr(), _stream(stream)))
    return Y, prof[:grid]


# ---------------------------------------------------------------------------
# expert-parallel bookkeeping kernels (include/moe_sm100_ep.h)
# ---------------------------------------------------------------------------
def moe_ep_dispatch_plan(topk_ids, E: int, G: int, stream=None):
    """-> counts2 [G, 2] (rows sent to d, result rows d returns), send_off [G+1], send_tok [G*T],
    send_meta [G*T, k] (device; only the first send_off[G] rows are meaningful)."""
    import torch

    T, k = topk_ids.shape
    dev = topk_ids.device
    counts2 = torch.empty((G, 2), dtype=torch.int32, device=dev)
    send_off = torch.empty(G + 1, dtype=torch.int32, device=dev)
    cap = max(G * T, 1)
    send_tok = torch.empty(cap, dtype=torch.int32, device=dev)
    send_meta = torch.empty((cap, k), dtype=torch.int32, device=dev)
    _check(lib().moe_ep_dispatch_plan(topk_ids.data_ptr(), T, k, E, G, counts2.data_ptr(), send_off.data_ptr(),
                                      send_tok.data_ptr(), send_meta.data_ptr(), _stream(stream)))
    return counts2, send_off, send_tok, send_meta


def moe_gather_rows(src, idx, out=None, stream=None):
    import torch

    n = int(idx.numel())
    if out is None:
        out = torch.empty((n,) + tuple(src.shape[1:]), dtype=src.dtype, device=src.device)
    row_bytes = src[0].numel() * src.element_size() if src.shape[0] else 16
    _check(lib().moe_gather_rows(src.data_ptr(), idx.data_ptr(), n, row_bytes, out.data_ptr(), _stream(stream)))
    return out


def moe_ep_combine_map(token_idx, slot, recv_off, ret_off, G: int, k: int, stream=None):
    import torch

    n = int(token_idx.numel())
    dev = token_idx.device
    cursor = torch.empty(G, dtype=torch.int32, device=dev)
    row_map = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    ret_meta = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    _check(lib().moe_ep_combine_map(token_idx.data_ptr(), slot.data_ptr(), n, recv_off.data_ptr(),
                                    ret_off.data_ptr(), G, k, cursor.data_ptr(), row_map.data_ptr(),
                                    ret_meta.data_ptr(), _stream(stream)))
    return row_map[:n], ret_meta[:n]


def moe_ep_unpack(rows, ret_meta, ret_off, send_off, send_tok, G: int, k: int, out, stream=None):
    n = int(rows.shape[0])
    row_bytes = rows[0].numel() * rows.element_size() if n else 16
    _check(lib().moe_ep_unpack(rows.data_ptr(), ret_meta.data_ptr(), n, ret_off.data_ptr(), send_off.data_ptr(),
                               send_tok.data_ptr(), G, k, row_bytes, out.data_ptr(), _stream(stream)))
    return out


def moe_decode_debug(plan: Plan, stream=None):
    import torch

    total = plan.total_tiles
    out = torch.full((max(total, 1), 5), -1, dtype=torch.int32, device="cuda")
    _check(lib().moe_decode_debug(plan.handle, out.data_ptr(), _stream(stream)))
    return out[:total]


def moe_probe_gather4(X, rows, col0: int, stream=None):
    import torch

    out = torch.zeros(16384, dtype=torch.uint8, device=X.device)
    _check(lib().moe_probe_gather4(X.data_ptr(), X.shape[0], X.shape[1], rows.data_ptr(), col0, out.data_ptr(),
                                   _stream(stream)))
    return out


def moe_forward(topk_ids, X, W, E: int, bm: int = 0, bn: int = 0, out_dtype=None, plan: Plan | None = None,
                stream=None, device_plan: bool = True, Y=None, scale=None):
    """One MoE expert-GEMM step: route -> plan -> single-launch GEMM.

    X / W in bf16 run moe_gemm; in FP8 E4M3 (torch.float8_e4m3fn or uint8 codes) moe_gemm_fp8 with
    the optional per-expert fp32 `scale`.

    device_plan=True: the plan is built on the device from the route's counts (moe_plan_device),
    no host synchronisation; counts are returned as a device tensor.  device_plan=False: counts
    are copied to the host and planned there (moe_plan_update; P:142's first option).
    Returns (Y, counts, row_off, token_idx, slot, plan)."""
    import torch

    H, N = int(X.shape[1]), int(W.shape[2])
    if device_plan:
        if plan is None:
            if bm == 0 and bn == 0:
                bm, bn = suggest_tile(topk_ids.numel(), E, H, N)
            plan = Plan(None, H, N, bm, bn, stream=stream, E=E)
        counts, row_off, token_idx, slot, _ = moe_route(topk_ids, E, stream=stream, plan=plan)
        counts_out = counts
    else:
        counts, row_off, token_idx, slot, _ = moe_route(topk_ids, E, stream=stream)
        counts_out = counts.cpu().numpy()
        if plan is None:
            plan = Plan(counts_out, H, N, bm, bn, stream=stream)
        else:
            plan.update(counts_out, stream=stream)
    if X.dtype in (torch.float8_e4m3fn, torch.uint8):
        Y = moe_gemm_fp8(plan, X, token_idx, W, scale, Y=Y, out_dtype=out_dtype or torch.bfloat16, stream=stream)
    else:
        Y = moe_gemm(plan, X, token_idx, W, Y=Y, out_dtype=out_dtype or torch.bfloat16, stream=stream)
    return Y, counts_out, row_off, token_idx, slot, plan


# ---------------------------------------------------------------------------
# the expert-parallel step in the library (include/moe_sm100_ep.h, moe_ep_*: NCCL from C++)
# ---------------------------------------------------------------------------
def moe_ep_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().moe_ep_unique_id(buf))
    return buf.raw


class NativeExpertParallel:
    """One rank of the library's expert-parallel step (moe_ep_create / moe_ep_forward).
    unique_id: 128 bytes from moe_ep_unique_id() on rank 0, shared by the caller."""

    def __init__(self, unique_id: bytes, rank: int, world: int, E: int, W_local, w_scale=None, bm: int = 0,
                 bn: int = 0, handle=None, fused: bool = True):
        import torch

        self.W, self.w_scale, self.E, self.world = W_local, w_scale, E, world
        self.fp8 = W_local.dtype in (torch.uint8, torch.float8_e4m3fn)
        assert W_local.is_cuda and W_local.is_contiguous() and W_local.dim() == 3
        assert W_local.shape[0] == E // world, "W_local must hold this rank's E / world experts"
        assert self.fp8 or W_local.dtype == torch.bfloat16
        if w_scale is not None:
            assert self.fp8 and w_scale.dtype == torch.float32 and w_scale.is_contiguous()
            assert w_scale.numel() == W_local.shape[0]
        if handle is not None:                     # from loopback_group (test transport)
            self._h = handle
            return
        assert len(unique_id) == 128
        self._h = ctypes.c_void_p()
        _check(lib().moe_ep_create(ctypes.create_string_buffer(unique_id, 128), rank, world, E, bm, bn,
                                   0 if fused else MOE_EP_UNFUSED, ctypes.byref(self._h)))

    @staticmethod
    def loopback_group(world: int, E: int, W_locals, w_scales=None, bm: int = 0, bn: int = 0, fused: bool = False):
        """`world` virtual ranks on one device exchanging by device copies (moe_ep_create_loopback,
        include/moe_sm100_debug.h); fused: the GEMM epilogue writes into the owners' buffers.
        Call each rank's forward from its own thread and stream."""
        hs = (ctypes.c_void_p * world)()
        _check(lib().moe_ep_create_loopback(world, E, bm, bn, 1 if fused else 0, hs))
        return [NativeExpertParallel(b"", r, world, E, W_locals[r], None if w_scales is None else w_scales[r],
                                     handle=ctypes.c_void_p(hs[r])) for r in range(world)]

    def forward(self, topk_local, X_local, out=None, out_dtype=None, stream=None):
        import torch

        out_dtype = out_dtype or torch.bfloat16
        T, k = topk_local.shape
        N = self.W.shape[2]
        assert X_local.is_contiguous() and topk_local.dtype == torch.int32 and topk_local.is_contiguous()
        assert X_local.dim() == 2 and X_local.shape[0] == T and X_local.shape[1] == self.W.shape[1], \
            "X_local must be [T, H] with the experts' H"
        x_fp8 = X_local.dtype in (torch.uint8, torch.float8_e4m3fn)
        assert x_fp8 == self.fp8 and (x_fp8 or X_local.dtype == torch.bfloat16), "X and W must both be bf16 or E4M3"
        if out is None:
            out = torch.empty((T * k, N), dtype=out_dtype, device=X_local.device)
        assert out.is_contiguous() and tuple(out.shape) == (T * k, N) and out.dtype in (torch.bfloat16, torch.float32)
        _check(lib().moe_ep_forward(self._h, topk_local.data_ptr(), T, k, X_local.data_ptr(), X_local.shape[1],
                                    MOE_DTYPE_E4M3 if self.fp8 else MOE_DTYPE_BF16, self.W.data_ptr(), N,
                                    self.w_scale.data_ptr() if self.w_scale is not None else None, out.data_ptr(),
                                    MOE_DTYPE_F32 if out.dtype == torch.float32 else MOE_DTYPE_BF16,
                                    _stream(stream)))
        return out

    def last_gemm_ms(self) -> float:
        """Device time of the last step's GEMM launch (0 when this rank had no local rows)."""
        ms = ctypes.c_float()
        _check(lib().moe_ep_last_gemm_ms(self._h, ctypes.byref(ms)))
        return float(ms.value)

    def last_rows(self):
        a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(lib().moe_ep_last_rows(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
        return {"sent": a.value, "received": b.value, "local_rows": c.value}

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.moe_ep_destroy(h)
            self._h = None


MOE_EP_PEER_BLOB_BYTES = 256


class PeerExpertParallel(NativeExpertParallel):
    """One rank of the library's expert-parallel step over symmetric peer memory (moe_ep_peer_create /
    moe_ep_peer_connect / moe_ep_forward; include/moe_sm100_ep.h): dispatch rows are stored straight into
    the owners' receive buffers and the GEMM epilogue stores result rows straight into the token owners'
    outputs (CUDA IPC mappings; NVLink stores between GPUs), ordered by device-side epoch flags.
    allgather(blob: bytes) -> list[bytes] in rank order is the caller's plumbing (e.g. torch.distributed
    all_gather_object); construct with connect=False and call connect(blobs) to drive several handles of
    one process (virtual ranks, see `group`)."""

    def __init__(self, rank: int, world: int, E: int, W_local, max_tokens: int, k: int, allgather=None,
                 w_scale=None, bm: int = 0, bn: int = 0, max_out_bytes: int | None = None, connect: bool = True):
        import torch

        super().__init__(b"", rank, world, E, W_local, w_scale=w_scale, handle=ctypes.c_void_p(0))
        H, N = W_local.shape[1], W_local.shape[2]
        x_row = H * (1 if self.fp8 else 2)
        y_row = max_out_bytes if max_out_bytes is not None else N * 4
        self.max_tokens, self.k = max_tokens, k
        self._h = ctypes.c_void_p()
        blob = ctypes.create_string_buffer(MOE_EP_PEER_BLOB_BYTES)
        _check(lib().moe_ep_peer_create(rank, world, E, bm, bn, max_tokens, k, x_row, y_row, ctypes.byref(self._h),
                                        blob))
        self.blob = blob.raw
        self._torch = torch
        if connect:
            assert allgather is not None, "allgather(blob) -> [blob of rank 0, ..., rank world-1] is needed"
            self.connect(allgather(self.blob))

    def connect(self, blobs):
        assert len(blobs) == self.world and all(len(b) == MOE_EP_PEER_BLOB_BYTES for b in blobs)
        _check(lib().moe_ep_peer_connect(self._h, ctypes.create_string_buffer(b"".join(blobs), len(blobs) *
                                                                                MOE_EP_PEER_BLOB_BYTES)))

    @staticmethod
    def group(world: int, E: int, W_locals, max_tokens: int, k: int, w_scales=None, bm: int = 0, bn: int = 0,
              max_out_bytes: int | None = None):
        """`world` virtual ranks of this process on the current device (one host thread can drive them
        all: a step never blocks the host)."""
        eps = [PeerExpertParallel(r, world, E, W_locals[r], max_tokens, k, w_scale=None if w_scales is None
                                  else w_scales[r], bm=bm, bn=bn, max_out_bytes=max_out_bytes, connect=False)
               for r in range(world)]
        blobs = [e.blob for e in eps]
        for e in eps:
            e.connect(blobs)
        return eps

    def output(self, T: int, N: int, dtype=None):
        """The handle's own output rows as a [T * k, N] tensor view (zero copy: pass it as `out`)."""
        torch = self._torch
        dtype = dtype or torch.bfloat16
        ptr, nbytes = ctypes.c_void_p(), ctypes.c_int64()
        _check(lib().moe_ep_peer_output(self._h, ctypes.byref(ptr), ctypes.byref(nbytes)))
        esz = torch.empty((), dtype=dtype).element_size()
        assert T * self.k * N * esz <= nbytes.value
        return _device_view(ptr.value, (T * self.k, N), dtype, torch.cuda.current_device())

    def set_timeout(self, seconds: float):
        _check(lib().moe_ep_peer_set_timeout(self._h, int(seconds * 1e9)))

    def status(self) -> int:
        """0, or 2 if a device-side wait of the last step timed out (synchronises)."""
        st = ctypes.c_int32()
        _check(lib().moe_ep_peer_status(self._h, ctypes.byref(st)))
        return int(st.value)


def _device_view(ptr: int, shape, dtype, device: int):
    """A torch tensor over library-owned device memory (no copy; the library keeps ownership)."""
    import torch

    class _Cai:
        pass

    typestr = {torch.bfloat16: "<i2", torch.float32: "<f4"}[dtype]
    c = _Cai()
    c.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False), "version": 3,
                                  "strides": None}
    t = torch.as_tensor(c, device=torch.device("cuda", device))
    return t.view(dtype) if dtype == torch.bfloat16 else t

