"""The paper's framework primitives as GPU ops, with the reference API
(/root/reference/pkg/src/seghull/segments.py, primitives.py):

  ScanSpec, segmented_scan, head_index_broadcast, segment_ids,
  reduce_broadcast                                   (segments.py:27-266)
  PermutationMap, flag_permute, compact, scatter     (primitives.py:26-176)

Inputs may be numpy arrays (copied to the current CUDA device; results come
back as numpy, like the reference) or CUDA tensors (results stay on the
device).  Every op runs in the C-ABI library's own kernels
(csrc/sh_prims.cuh); there is no CPU fallback.  Validation and error
messages follow the reference (ContractViolation).
"""

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import ContractViolation

OPERATORS = ("sum", "max", "min")
DIRECTIONS = ("forward", "backward")
MODES = ("inclusive", "exclusive")
_OP = {"sum": 0, "max": 1, "min": 2}


@dataclass(frozen=True)
class ScanSpec:
    """Operator in {sum, max, min}, direction, mode (segments.py:27-49)."""

    operator: str
    direction: str = "forward"
    mode: str = "inclusive"

    def __post_init__(self):
        if self.operator not in OPERATORS:
            raise ValueError(f"unknown operator {self.operator!r}")
        if self.direction not in DIRECTIONS:
            raise ValueError(f"unknown direction {self.direction!r}")
        if self.mode not in MODES:
            raise ValueError(f"unknown mode {self.mode!r}")


@dataclass(frozen=True)
class PermutationMap:
    """Destination index per element (primitives.py:26-38)."""

    p: object
    out_len: int


def _device():
    return torch.device("cuda", torch.cuda.current_device())


def _to_dev(a, dtype):
    """-> (contiguous CUDA tensor of dtype, True if the input was numpy)."""
    if torch.is_tensor(a):
        if not a.is_cuda:
            return a.to(_device(), dtype=dtype).contiguous(), True
        return a.to(dtype=dtype).contiguous(), False
    return torch.from_numpy(np.ascontiguousarray(a)).to(_device(), dtype=dtype), True


def _out(t, host):
    return t.cpu().numpy() if host else t


def _heads(s, n=None):
    """Reference as_segment_flags/validate_segments (segments.py:64-87)."""
    if torch.is_tensor(s):
        if s.dim() != 1:
            raise ContractViolation(f"segment flags must be one-dimensional, got shape {tuple(s.shape)}")
        size = s.numel()
    else:
        s = np.ascontiguousarray(s, dtype=bool)
        if s.ndim != 1:
            raise ContractViolation(f"segment flags must be one-dimensional, got shape {s.shape}")
        size = s.size
    want = size if n is None else n
    if size != want:
        raise ContractViolation(f"segment flags have length {size}, expected {want}")
    h, host = _to_dev(s, torch.uint8)
    if size and not bool(h[0].item()):
        raise ContractViolation("first element is not a segment head")
    return h, host


def _call(rc):
    if rc != _lib.SH_OK:
        if rc == _lib.SH_CONTRACT:
            raise ContractViolation(_lib.last_error())
        raise RuntimeError(f"seghull_b200 error {rc}: {_lib.last_error()}")


def _ctx():
    dev = torch.cuda.current_device()
    return _lib.context(dev), torch.cuda.current_stream().cuda_stream


def segmented_scan(values, s, spec):
    """Run ``spec`` inside every segment (segments.py:201-234)."""
    if not isinstance(spec, ScanSpec):
        spec = ScanSpec(*spec)
    is_t = torch.is_tensor(values)
    arr = values if is_t else np.asarray(values)
    dt = arr.dtype
    floating = dt.is_floating_point if is_t else np.issubdtype(dt, np.floating)
    boolish = (dt == torch.bool) if is_t else (dt == bool)
    integer = (not floating) and (boolish or (not dt.is_complex if is_t else np.issubdtype(dt, np.integer)))
    if (arr.dim() if is_t else arr.ndim) != 1:
        raise ContractViolation("values must be one-dimensional")
    if floating and spec.operator == "sum":
        raise ContractViolation(
            "sum scans are integer-only (float accumulation order would break the determinism "
            "contract); cast or use max/min")
    if not floating and not integer:
        raise ContractViolation(f"unsupported value dtype {dt}")
    n = arr.numel() if is_t else arr.size
    heads, _ = _heads(s, n)
    v, host = _to_dev(arr, torch.float64 if floating else torch.int64)
    out = torch.empty_like(v)
    if n:
        ctx, st = _ctx()
        _call(_lib.lib().sh_segmented_scan(ctx, v.data_ptr(), 1 if floating else 0, heads.data_ptr(), n,
                                           _OP[spec.operator], spec.direction == "backward",
                                           spec.mode == "exclusive", out.data_ptr(), st))
    return _out(out, host)


def head_index_broadcast(s):
    """Index of the owning segment's head (segments.py:237-247)."""
    heads, host = _heads(s)
    idx = torch.arange(heads.numel(), dtype=torch.int64, device=heads.device)
    seeded = torch.where(heads.bool(), idx, torch.zeros_like(idx))
    return _out(segmented_scan(seeded, heads, ScanSpec("sum")), host)


def segment_ids(s):
    """0-based segment number per element (segments.py:250-253)."""
    heads, host = _heads(s)
    n = heads.numel()
    one = torch.zeros(n, dtype=torch.uint8, device=heads.device)
    if n:
        one[0] = 1
    r = segmented_scan(heads.to(torch.int64), one, ScanSpec("sum")) - 1
    return _out(r, host)


def reduce_broadcast(values, s, operator):
    """Whole-segment reduction broadcast to every element (segments.py:256-266)."""
    inclusive = segmented_scan(values, s, ScanSpec(operator, "forward", "inclusive"))
    back = "min" if operator == "min" else "max"
    return segmented_scan(inclusive, s, ScanSpec(back, "backward", "inclusive"))


def flag_permute(f, s, k):
    """Stable in-segment grouping by state (primitives.py:91-117)."""
    if k < 1:
        raise ContractViolation(f"state count must be >= 1, got {k}")
    fa, host = _to_dev(f, torch.int64)
    if fa.dim() != 1:
        raise ContractViolation("state flags must be one-dimensional")
    n = fa.numel()
    heads, _ = _heads(s)
    if heads.numel() != n:
        raise ContractViolation(f"state flags have length {n} but segment flags {heads.numel()}")
    if n and (int(fa.min()) < 0 or int(fa.max()) >= k):
        raise ContractViolation(f"state flags must lie in [0, {k}), got range [{int(fa.min())}, {int(fa.max())}]")
    p = torch.empty(n, dtype=torch.int64, device=fa.device)
    s_new = torch.empty(n, dtype=torch.uint8, device=fa.device)
    if n:
        ctx, st = _ctx()
        _call(_lib.lib().sh_flag_permute(ctx, fa.data_ptr(), heads.data_ptr(), n, k, p.data_ptr(),
                                         s_new.data_ptr(), st))
    return PermutationMap(_out(p, host), n), _out(s_new.bool(), host)


def compact(b, s):
    """Remove false-flagged elements, preserving order (primitives.py:120-148)."""
    ba, host = _to_dev(b, torch.uint8)
    heads, _ = _heads(s)
    n = ba.numel()
    if ba.dim() != 1 or n != heads.numel():
        raise ContractViolation(f"mask has length {n} but segment flags {heads.numel()}")
    p = torch.empty(n, dtype=torch.int64, device=ba.device)
    s_new = torch.zeros(max(n, 1), dtype=torch.uint8, device=ba.device)
    out_len = ctypes.c_int64(0)
    if n:
        ctx, st = _ctx()
        _call(_lib.lib().sh_compact(ctx, (ba != 0).to(torch.uint8).data_ptr(), heads.data_ptr(), n,
                                    p.data_ptr(), ctypes.byref(out_len), s_new.data_ptr(), st))
    m = int(out_len.value)
    return PermutationMap(_out(p, host), m), _out(s_new[:m].bool(), host)


def scatter(data, pm, live=None):
    """out[p[i]] = data[i] for live i, with collision / range checks
    (primitives.py:151-176)."""
    is_t = torch.is_tensor(data)
    d, host = (data.contiguous(), not data.is_cuda) if is_t else (torch.from_numpy(np.ascontiguousarray(data)), True)
    pa, _ = _to_dev(pm.p, torch.int64)
    if d.shape[0] != pa.numel():
        raise ContractViolation(f"data has length {d.shape[0]} but map {pa.numel()}")
    lv = None
    if live is not None:
        lv, _ = _to_dev(live, torch.uint8)
        if lv.numel() != pa.numel():
            raise ContractViolation("live mask length does not match map")
    d = d.to(_device())
    out = torch.empty((pm.out_len,) + tuple(d.shape[1:]), dtype=d.dtype, device=d.device)
    row = d.element_size() * (int(np.prod(d.shape[1:])) if d.dim() > 1 else 1)
    ctx, st = _ctx()
    _call(_lib.lib().sh_scatter(ctx, d.data_ptr(), row, pa.data_ptr(), lv.data_ptr() if lv is not None else None,
                                pa.numel(), pm.out_len, out.data_ptr() if pm.out_len else None, st))
    return out.cpu().numpy() if host else out
