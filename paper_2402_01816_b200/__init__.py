"""Thin Python binding of the C-ABI in ``include/gns.h`` (``libgns.so``).

Argument marshalling only: every step of the sort runs in the CUDA kernels of
``csrc/``.  There is no CPU fallback — importing this package without the
built library raises, and every call with a non-OK status raises
:class:`GnsError`.

Names mirror the C entry points (``gns_sort_f64`` ...).  Each takes torch CUDA
tensors (memory and streams are PyTorch's; the work is ours) and enqueues on
``torch.cuda.current_stream()`` unless a stream is given.  Convenience:
:func:`sort_` sorts ``keys`` (and ``vals``) in place.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

_HERE = os.path.dirname(os.path.abspath(__file__))
# GNS_LIB selects another build of the same library in this directory (e.g.
# libgns_debug.so, the bounds-asserting build); default libgns.so.
LIB_PATH = os.path.join(_HERE, os.environ.get("GNS_LIB", "libgns.so"))

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `make` or `python -c 'import __graft_entry__ as g; g.build()'`. "
        "There is no CPU fallback.")

_lib = ctypes.CDLL(LIB_PATH)

GNS_OK = 0
STATUS = {
    0: "GNS_OK", 1: "GNS_ERR_INVALID_ARGUMENT", 2: "GNS_ERR_UNSUPPORTED_FRACTION",
    3: "GNS_ERR_OUT_OF_MEMORY", 4: "GNS_ERR_CUDA", 5: "GNS_ERR_WORKSPACE_TOO_SMALL",
    6: "GNS_ERR_MISALIGNED",
}

_vp = ctypes.c_void_p
_sz = ctypes.c_size_t
_d = ctypes.c_double
_i = ctypes.c_int


class gns_plan_info(ctypes.Structure):
    _fields_ = [("tile", ctypes.c_int), ("merge_tile", ctypes.c_int),
                ("merge_passes", ctypes.c_int), ("hbm_passes", ctypes.c_int),
                ("launches", ctypes.c_int), ("element_passes", ctypes.c_double),
                ("left_len", _sz), ("workspace_bytes", _sz), ("buffer_elems", _sz),
                ("bytes_lower_bound", _sz)]


def _sig(name, argtypes, restype=ctypes.c_int):
    f = getattr(_lib, name)
    f.argtypes = argtypes
    f.restype = restype
    return f


_c = {
    "gns_sort_f64": _sig("gns_sort_f64", [_vp, _sz, _d, _vp]),
    "gns_sort_pairs_f64_u32": _sig("gns_sort_pairs_f64_u32", [_vp, _vp, _sz, _d, _vp]),
    "gns_workspace_bytes": _sig("gns_workspace_bytes", [_sz, _d, _i], _sz),
    "gns_sort_f64_ws": _sig("gns_sort_f64_ws", [_vp, _sz, _d, _vp, _sz, _vp]),
    "gns_sort_pairs_f64_u32_ws": _sig("gns_sort_pairs_f64_u32_ws", [_vp, _vp, _sz, _d, _vp, _sz, _vp]),
    "gns_sort_target_f64": _sig("gns_sort_target_f64", [_vp, _vp, _sz, _d, _i, _vp, _sz, _vp]),
    "gns_sort_keys": _sig("gns_sort_keys", [_vp, _i, _vp, _sz, _d, _i, _vp, _sz, _vp]),
    "gns_sort_omit": _sig("gns_sort_omit", [_vp, _i, _vp, _sz, _i, _vp, _sz, _vp]),
    "gns_sort_keys_u64": _sig("gns_sort_keys_u64", [_vp, _i, _vp, _sz, _i, _vp, _sz, _vp]),
    "gns_workspace_bytes_u64": _sig("gns_workspace_bytes_u64", [_sz], _sz),
    "gns_sort_f32": _sig("gns_sort_f32", [_vp, _vp, _sz, _i, _vp, _sz, _vp]),
    "gns_workspace_bytes_f32": _sig("gns_workspace_bytes_f32", [_sz, _i], _sz),
    "gns_split_cuts": _sig("gns_split_cuts", [_vp, _i, _sz, _vp, _vp, _vp, _i, _i, _vp, _vp]),
    "gns_merge_two": _sig("gns_merge_two", [_vp, _vp, _sz, _vp, _vp, _sz, _vp, _vp, _i, _vp]),
    "gns_plan": _sig("gns_plan", [_sz, _d, _i, ctypes.POINTER(gns_plan_info)]),
    "gns_tile_sort": _sig("gns_tile_sort", [_vp, _vp, _vp, _vp, _sz, _vp]),
    "gns_merge_workspace_bytes": _sig("gns_merge_workspace_bytes", [_sz], _sz),
    "gns_merge_pass": _sig("gns_merge_pass", [_vp, _vp, _vp, _vp, _sz, _sz, _vp, _sz, _vp]),
    "gns_merge_inplace_top": _sig("gns_merge_inplace_top", [_vp, _vp, _vp, _vp, _sz, _sz, _vp, _sz, _vp]),
    "gns_timing_begin": _sig("gns_timing_begin", [_i]),
    "gns_pool_high_water": _sig("gns_pool_high_water", [_i], _sz),
    "gns_timing_end": _sig("gns_timing_end", [ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_int), _i]),
    "gns_tile_elems": _sig("gns_tile_elems", []),
    "gns_merge_tile_elems": _sig("gns_merge_tile_elems", []),
    "gns_status_string": _sig("gns_status_string", [_i], ctypes.c_char_p),
    "gns_last_error_string": _sig("gns_last_error_string", [], ctypes.c_char_p),
}

EXPORTED = tuple(_c)


class GnsError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = _c["gns_last_error_string"]().decode(errors="replace")
        super().__init__(f"{where}: {STATUS.get(status, status)}: {msg}")


def _check(rc: int, where: str) -> None:
    if rc != GNS_OK:
        raise GnsError(rc, where)


# ----------------------------------------------------------- raw-pointer layer
# The C names, taking integers (device pointers, sizes, a cudaStream_t handle).

def gns_sort_f64(keys_ptr: int, n: int, buffer_fraction: float, stream: int) -> int:
    return _c["gns_sort_f64"](keys_ptr, n, buffer_fraction, stream)


def gns_sort_pairs_f64_u32(keys_ptr: int, vals_ptr: int, n: int, buffer_fraction: float, stream: int) -> int:
    return _c["gns_sort_pairs_f64_u32"](keys_ptr, vals_ptr, n, buffer_fraction, stream)


def gns_workspace_bytes(n: int, buffer_fraction: float, with_vals: bool) -> int:
    return _c["gns_workspace_bytes"](n, buffer_fraction, int(bool(with_vals)))


def gns_sort_f64_ws(keys_ptr, n, buffer_fraction, ws_ptr, ws_bytes, stream) -> int:
    return _c["gns_sort_f64_ws"](keys_ptr, n, buffer_fraction, ws_ptr, ws_bytes, stream)


def gns_sort_pairs_f64_u32_ws(keys_ptr, vals_ptr, n, buffer_fraction, ws_ptr, ws_bytes, stream) -> int:
    return _c["gns_sort_pairs_f64_u32_ws"](keys_ptr, vals_ptr, n, buffer_fraction, ws_ptr, ws_bytes, stream)


TARGETS = {"AscLeft": 0, "AscRight": 1, "DescLeft": 2, "DescRight": 3}


def gns_sort_target_f64(keys_ptr, vals_ptr, n, buffer_fraction, target, ws_ptr, ws_bytes, stream) -> int:
    return _c["gns_sort_target_f64"](keys_ptr, vals_ptr, n, buffer_fraction, target, ws_ptr, ws_bytes, stream)


KEY_TYPES = {"f64": 0, "i64": 1, "u64": 2}


def gns_sort_keys(keys_ptr, key_type, vals_ptr, n, buffer_fraction, target, ws_ptr, ws_bytes, stream) -> int:
    return _c["gns_sort_keys"](keys_ptr, key_type, vals_ptr, n, buffer_fraction, target, ws_ptr, ws_bytes, stream)


def gns_sort_keys_u64(keys_ptr, key_type, vals_ptr, n, target, ws_ptr, ws_bytes, stream) -> int:
    return _c["gns_sort_keys_u64"](keys_ptr, key_type, vals_ptr, n, target, ws_ptr, ws_bytes, stream)


def gns_workspace_bytes_u64(n) -> int:
    return _c["gns_workspace_bytes_u64"](n)


def gns_sort_f32(keys_ptr, vals_ptr, n, target, ws_ptr, ws_bytes, stream) -> int:
    return _c["gns_sort_f32"](keys_ptr, vals_ptr, n, target, ws_ptr, ws_bytes, stream)


def gns_workspace_bytes_f32(n, with_vals) -> int:
    return _c["gns_workspace_bytes_f32"](n, with_vals)


def gns_sort_omit(keys_ptr, key_type, vals_ptr, n, target, ws_ptr, ws_bytes, stream) -> int:
    return _c["gns_sort_omit"](keys_ptr, key_type, vals_ptr, n, target, ws_ptr, ws_bytes, stream)


def gns_split_cuts(keys_ptr, key_type, n, spl_keys, spl_rank, spl_pos, nsplit, my_rank, cuts, stream) -> int:
    return _c["gns_split_cuts"](keys_ptr, key_type, n, spl_keys, spl_rank, spl_pos, nsplit, my_rank, cuts, stream)


def gns_merge_two(a_k, a_v, la, b_k, b_v, lb, dst_k, dst_v, key_type, stream) -> int:
    return _c["gns_merge_two"](a_k, a_v, la, b_k, b_v, lb, dst_k, dst_v, key_type, stream)


def gns_plan(n: int, buffer_fraction: float, with_vals: bool) -> gns_plan_info:
    info = gns_plan_info()
    _check(_c["gns_plan"](n, buffer_fraction, int(bool(with_vals)), ctypes.byref(info)), "gns_plan")
    return info


def gns_tile_sort(src_k, src_v, dst_k, dst_v, n, stream) -> int:
    return _c["gns_tile_sort"](src_k, src_v, dst_k, dst_v, n, stream)


def gns_merge_workspace_bytes(n: int) -> int:
    return _c["gns_merge_workspace_bytes"](n)


def gns_merge_pass(src_k, src_v, dst_k, dst_v, n, run_len, ws, ws_bytes, stream) -> int:
    return _c["gns_merge_pass"](src_k, src_v, dst_k, dst_v, n, run_len, ws, ws_bytes, stream)


def gns_merge_inplace_top(keys, vals, left_k, left_v, nl, n, ws, ws_bytes, stream) -> int:
    return _c["gns_merge_inplace_top"](keys, vals, left_k, left_v, nl, n, ws, ws_bytes, stream)


def gns_pool_high_water(reset: int) -> int:
    return _c["gns_pool_high_water"](reset)


def gns_timing_begin(max_launches: int) -> int:
    return _c["gns_timing_begin"](max_launches)


def gns_timing_end(cap: int = 4096):
    """Returns [(kind, ms), ...] of the launches timed since gns_timing_begin."""
    ms = (ctypes.c_float * cap)()
    kind = (ctypes.c_int * cap)()
    n = _c["gns_timing_end"](ms, kind, cap)
    if n < 0:
        raise GnsError(GNS_OK, "gns_timing_end")
    return [(kind[i], ms[i]) for i in range(min(n, cap))]


LAUNCH_KINDS = {1: "tile_sort", 2: "merge_pass", 3: "partition", 4: "inplace_deps", 5: "inplace_merge", 6: "reverse",
                7: "split_cuts", 8: "gather_samples", 9: "omit_plan", 10: "omit_prep", 11: "omit_final",
                12: "iota", 13: "gather_u64", 14: "f32_tile_sort", 15: "f32_merge", 16: "f32_reverse",
                17: "f32_partition", 18: "merge_multi", 19: "peel_head", 20: "peel_merge", 21: "small_sort",
                22: "rank4", 23: "merge4"}


def gns_tile_elems() -> int:
    return _c["gns_tile_elems"]()


def gns_merge_tile_elems() -> int:
    return _c["gns_merge_tile_elems"]()


def gns_status_string(s: int) -> str:
    return _c["gns_status_string"](s).decode()


def gns_last_error_string() -> str:
    return _c["gns_last_error_string"]().decode(errors="replace")


# --------------------------------------------------------------- torch layer

def _stream_handle(stream) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    return int(t.data_ptr())


def _key_type(keys) -> int:
    import torch
    kt = {torch.float64: 0, torch.int64: 1, torch.uint64: 2}.get(keys.dtype)
    if kt is None:
        raise TypeError("keys must be float64, int64 or uint64")
    return kt


def _check_keys(keys, vals, any_key_type: bool = False):
    import torch
    if any_key_type:
        _key_type(keys)
    elif keys.dtype != torch.float64:
        raise TypeError("keys must be a contiguous CUDA float64 tensor")
    if not keys.is_cuda or not keys.is_contiguous():
        raise TypeError("keys must be a contiguous CUDA tensor")
    if vals is not None:
        if vals.dtype != torch.uint32 or not vals.is_cuda or not vals.is_contiguous():
            raise TypeError("vals must be a contiguous CUDA uint32 tensor")
        if vals.numel() != keys.numel():
            raise ValueError("keys and vals differ in length")


def sort_u64_(keys, vals, workspace=None, stream=None, target: str = "AscLeft"):
    """NEXT f3: stable sort of ``keys`` (float64 / int64 / uint64) moving a
    64-bit payload ``vals`` (uint64 or int64, contiguous CUDA) with each key
    (gns_sort_keys_u64, full buffer).  ``workspace``: optional uint8 CUDA
    tensor of >= workspace_bytes_u64(n) bytes."""
    _check_keys(keys, None, any_key_type=True)
    import torch
    if vals.dtype not in (torch.uint64, torch.int64) or not vals.is_cuda or not vals.is_contiguous():
        raise TypeError("vals must be a contiguous CUDA uint64/int64 tensor")
    if vals.numel() != keys.numel():
        raise ValueError("keys and vals differ in length")
    n = keys.numel()
    wp = _ptr(workspace) if workspace is not None else None
    wb = workspace.numel() * workspace.element_size() if workspace is not None else 0
    _check(gns_sort_keys_u64(_ptr(keys), _key_type(keys), _ptr(vals), n, TARGETS[target], wp, wb,
                             _stream_handle(stream)), "sort_u64_")
    return keys, vals


def workspace_bytes_u64(n: int) -> int:
    return gns_workspace_bytes_u64(n)


def sort_f32_(keys, vals=None, workspace=None, stream=None, target: str = "AscLeft"):
    """NEXT f3: stable sort of float32 ``keys`` (and uint32 ``vals``) on the
    GPU (gns_sort_f32: the 4-byte kernel set, full buffer, %RAM 2.0).
    ``workspace``: optional uint8 CUDA tensor of >= workspace_bytes_f32(n,
    vals is not None) bytes."""
    import torch
    if keys.dtype != torch.float32 or not keys.is_cuda or not keys.is_contiguous():
        raise TypeError("keys must be a contiguous CUDA float32 tensor")
    if vals is not None:
        if vals.dtype != torch.uint32 or not vals.is_cuda or not vals.is_contiguous():
            raise TypeError("vals must be a contiguous CUDA uint32 tensor")
        if vals.numel() != keys.numel():
            raise ValueError("keys and vals differ in length")
    n = keys.numel()
    wp = _ptr(workspace) if workspace is not None else None
    wb = workspace.numel() * workspace.element_size() if workspace is not None else 0
    _check(gns_sort_f32(_ptr(keys), _ptr(vals), n, TARGETS[target], wp, wb, _stream_handle(stream)), "sort_f32_")
    return keys, vals


def workspace_bytes_f32(n: int, with_vals: bool = False) -> int:
    return gns_workspace_bytes_f32(n, 1 if with_vals else 0)


def sort_omit_(keys, vals=None, workspace=None, stream=None, target: str = "AscLeft"):
    """NEXT f2 Omitsort schedule (gns_sort_omit): the same stable sort as
    ``sort_`` with the full buffer, but runs carry their location, merges of
    non-overlapping runs are omitted and presorted input moves no key.
    ``workspace``: optional uint8 CUDA tensor of >= workspace_bytes(n, 1.0,
    vals is not None) bytes."""
    _check_keys(keys, vals, any_key_type=True)
    n = keys.numel()
    wp = _ptr(workspace) if workspace is not None else None
    wb = workspace.numel() * workspace.element_size() if workspace is not None else 0
    _check(gns_sort_omit(_ptr(keys), _key_type(keys), _ptr(vals), n, TARGETS[target], wp, wb,
                         _stream_handle(stream)), "sort_omit_")
    return keys, vals


def sort_(keys, vals=None, buffer_fraction: float = 1.0, workspace=None, stream=None, target: str = "AscLeft"):
    """Stable in-place sort of ``keys`` (and ``vals``) on the GPU; ascending
    with ties in input order unless ``target`` names another of the four API
    targets (AscLeft, AscRight, DescLeft, DescRight).

    ``keys``: float64, int64 or uint64 (NEXT f3 key types, via gns_sort_keys).
    ``workspace``: optional uint8 CUDA tensor of >= workspace_bytes(...) bytes;
    without it the library allocates its buffer stream-ordered."""
    _check_keys(keys, vals, any_key_type=True)
    n = keys.numel()
    st = _stream_handle(stream)
    kt = _key_type(keys)
    if kt != 0:
        wp = _ptr(workspace) if workspace is not None else None
        wb = workspace.numel() * workspace.element_size() if workspace is not None else 0
        _check(gns_sort_keys(_ptr(keys), kt, _ptr(vals), n, buffer_fraction, TARGETS[target], wp, wb, st), "sort_")
        return keys, vals
    if target != "AscLeft":
        wp = _ptr(workspace) if workspace is not None else None
        wb = workspace.numel() * workspace.element_size() if workspace is not None else 0
        _check(gns_sort_target_f64(_ptr(keys), _ptr(vals), n, buffer_fraction, TARGETS[target], wp, wb, st),
               "sort_")
        return keys, vals
    if workspace is None:
        if vals is None:
            rc = gns_sort_f64(_ptr(keys), n, buffer_fraction, st)
        else:
            rc = gns_sort_pairs_f64_u32(_ptr(keys), _ptr(vals), n, buffer_fraction, st)
    else:
        wb = workspace.numel() * workspace.element_size()
        if vals is None:
            rc = gns_sort_f64_ws(_ptr(keys), n, buffer_fraction, _ptr(workspace), wb, st)
        else:
            rc = gns_sort_pairs_f64_u32_ws(_ptr(keys), _ptr(vals), n, buffer_fraction, _ptr(workspace), wb, st)
    _check(rc, "sort_")
    return keys, vals


def merge_two(a_k, a_v, b_k, b_v, stream=None, out=None):
    """Stable merge of two sorted runs (a wins ties) (gns_merge_two) into new
    tensors, or into ``out`` = (keys, vals-or-None) views of la + lb elements
    at natural alignment (the distributed sort's ping-pong tree).  Keys
    float64 / int64 / uint64; vals uint32 or None."""
    import torch
    kt = _key_type(a_k)
    if b_k.dtype != a_k.dtype:
        raise TypeError("a and b keys differ in dtype")
    la, lb = a_k.numel(), b_k.numel()
    if out is None:
        out_k = torch.empty(la + lb, dtype=a_k.dtype, device=a_k.device)
        out_v = None if a_v is None else torch.empty(la + lb, dtype=torch.uint32, device=a_k.device)
    else:
        out_k, out_v = out
        if out_k.numel() != la + lb or out_k.dtype != a_k.dtype or not out_k.is_contiguous():
            raise ValueError("out keys: a contiguous tensor of la + lb keys of the same dtype")
    _check(gns_merge_two(_ptr(a_k), _ptr(a_v), la, _ptr(b_k), _ptr(b_v), lb, _ptr(out_k), _ptr(out_v), kt,
                         _stream_handle(stream)), "merge_two")
    return out_k, out_v


def split_cuts(sorted_keys, spl_keys, spl_rank, spl_pos, my_rank: int, stream=None):
    """gns_split_cuts: int64 tensor of cut positions of this rank's sorted
    shard at the splitters (device tensors; spl_rank int32, spl_pos int64)."""
    import torch
    kt = _key_type(sorted_keys)
    k = spl_keys.numel()
    cuts = torch.empty(k, dtype=torch.int64, device=sorted_keys.device)
    _check(gns_split_cuts(_ptr(sorted_keys), kt, sorted_keys.numel(), _ptr(spl_keys), _ptr(spl_rank),
                          _ptr(spl_pos), k, my_rank, _ptr(cuts), _stream_handle(stream)), "split_cuts")
    return cuts


def workspace_bytes(n: int, buffer_fraction: float = 1.0, with_vals: bool = False) -> int:
    return gns_workspace_bytes(n, buffer_fraction, with_vals)


def alloc_workspace(n: int, buffer_fraction: float = 1.0, with_vals: bool = False, device="cuda"):
    import torch
    return torch.empty(max(1, workspace_bytes(n, buffer_fraction, with_vals)), dtype=torch.uint8, device=device)


def tile_sort(src_k, src_v=None, dst_k=None, dst_v=None, stream=None):
    """Row a2: sort each gns_tile_elems() tile of src into dst (default: in place)."""
    _check_keys(src_k, src_v)
    dst_k = src_k if dst_k is None else dst_k
    dst_v = src_v if dst_v is None else dst_v
    _check(gns_tile_sort(_ptr(src_k), _ptr(src_v), _ptr(dst_k), _ptr(dst_v), src_k.numel(),
                         _stream_handle(stream)), "tile_sort")
    return dst_k, dst_v


def merge_pass(src_k, src_v, dst_k, dst_v, run_len: int, workspace, stream=None):
    """Rows a3+a4: one merge level over runs of ``run_len`` (src -> dst)."""
    _check_keys(src_k, src_v)
    wb = workspace.numel() * workspace.element_size()
    _check(gns_merge_pass(_ptr(src_k), _ptr(src_v), _ptr(dst_k), _ptr(dst_v), src_k.numel(), run_len,
                          _ptr(workspace), wb, _stream_handle(stream)), "merge_pass")
    return dst_k, dst_v


def merge_inplace_top(keys, vals, left_k, left_v, nl: int, workspace, stream=None):
    """Row a6: merge left_k[0:nl) (buffer) with keys[nl:n) into keys[0:n)."""
    _check_keys(keys, vals)
    wb = workspace.numel() * workspace.element_size()
    _check(gns_merge_inplace_top(_ptr(keys), _ptr(vals), _ptr(left_k), _ptr(left_v), nl, keys.numel(),
                                 _ptr(workspace), wb, _stream_handle(stream)), "merge_inplace_top")
    return keys, vals


def plan(n: int, buffer_fraction: float = 1.0, with_vals: bool = False) -> dict:
    p = gns_plan(n, buffer_fraction, with_vals)
    return {f: getattr(p, f) for f, _ in gns_plan_info._fields_}
