"""Point sources on the device: PTS1 files straight into HBM and device-side
generation of the uniform-box clouds.

Mirrors the reference's point-file module
(/root/reference/pkg/src/seghull/pointfile.py):

  PTS1 binary: magic b"PTS1", dim uint32 LE, count uint64 LE (struct
  "<4sIQ", :20-21), then count*dim float64 LE point-major (:81-97)
  read_points_binary / write_points_binary / read_points / write_points
  PointFileError(ValueError) with the reference's messages

The device reader returns the payload as an (n, dim) float64 CUDA tensor in
the file's own point-major layout, which the hull entry points take as is
(row stride dim), so there is no transpose: the file is read in chunks into
two alternating pinned buffers while the previous chunk is copied to the
GPU, overlapping disk and PCIe.  CSV files (the reference's other format)
are parsed on the host with the reference's rules and copied.
"""

import os
import struct

import numpy as np
import torch

from . import _lib
from .geometry import PointSet

_MAGIC = b"PTS1"
_HEADER = struct.Struct("<4sIQ")
_CHUNK = 64 << 20  # bytes per pinned staging buffer


class PointFileError(ValueError):
    """Unreadable, corrupt, or inconsistent point file (pointfile.py:24-25)."""


def read_header(path):
    """(dim, count) of a PTS1 file, validated like read_points_binary
    (pointfile.py:81-97) without reading the payload."""
    try:
        size = os.path.getsize(path)
        with open(path, "rb") as fh:
            head = fh.read(_HEADER.size)
    except OSError as exc:
        raise PointFileError(f"{path}: {exc}") from None
    if len(head) < _HEADER.size:
        raise PointFileError(f"{path}: truncated header")
    magic, dim, count = _HEADER.unpack(head)
    if magic != _MAGIC:
        raise PointFileError(f"{path}: bad magic {magic!r}")
    if dim not in (2, 3):
        raise PointFileError(f"{path}: dim must be 2 or 3, got {dim}")
    expected = _HEADER.size + 8 * dim * count
    if size != expected:
        raise PointFileError(f"{path}: payload is {size} bytes, expected {expected}")
    return dim, count


def read_points_binary_device(path, device=None):
    """PTS1 file -> (n, dim) float64 tensor on ``device`` (default: the
    current CUDA device), read in pinned chunks overlapped with the H2D
    copies.  Empty files give a (0, dim) tensor."""
    dim, count = read_header(path)
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    out = torch.empty((count, dim), dtype=torch.float64, device=dev)
    if count == 0:
        return out
    flat = out.view(torch.uint8).view(-1)
    total = 8 * dim * count
    stream = torch.cuda.current_stream(dev)
    bufs = [torch.empty(min(_CHUNK, total), dtype=torch.uint8).pin_memory() for _ in range(2)]
    done = [None, None]
    with open(path, "rb", buffering=0) as fh:
        fh.seek(_HEADER.size)
        off, k = 0, 0
        while off < total:
            n = min(_CHUNK, total - off)
            b = bufs[k & 1]
            if done[k & 1] is not None:
                done[k & 1].synchronize()  # the copy out of this buffer has finished
            got = fh.readinto(memoryview(b.numpy())[:n])
            if got != n:
                raise PointFileError(f"{path}: short read at byte {_HEADER.size + off}")
            with torch.cuda.stream(stream):
                flat[off:off + n].copy_(b[:n], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(stream)
            done[k & 1] = ev
            off += n
            k += 1
    return out


def write_points_binary(path, points):
    """PointSet, (n, dim) tensor/array or tuple of columns -> PTS1 file
    (pointfile.py:74-78)."""
    if isinstance(points, PointSet):
        rows = points.as_rows()
    elif isinstance(points, (tuple, list)):
        rows = np.column_stack([c.cpu().numpy() if torch.is_tensor(c) else np.asarray(c) for c in points])
    else:
        rows = points.cpu().numpy() if torch.is_tensor(points) else np.asarray(points)
    rows = np.ascontiguousarray(rows, dtype="<f8")
    if rows.ndim != 2 or rows.shape[1] not in (2, 3):
        raise PointFileError("points must be 2D or 3D")
    with open(path, "wb") as fh:
        fh.write(_HEADER.pack(_MAGIC, rows.shape[1], rows.shape[0]))
        fh.write(rows.tobytes())


def read_points_csv(path) -> PointSet:
    """Reference CSV rules (pointfile.py:37-67): optional '# x,y[,z]' first
    line, 2 or 3 columns, consistent column count."""
    cols = None
    header_cols = None
    data = []
    try:
        fh = open(path)
    except OSError as exc:
        raise PointFileError(f"{path}: {exc}") from None
    with fh:
        for lineno, line in enumerate(fh, start=1):
            line = line.strip()
            if not line:
                continue
            if line.startswith("#"):
                if lineno == 1:
                    label = line.lstrip("#").strip()
                    if label in ("x,y", "x,y,z"):
                        header_cols = label.count(",") + 1
                    continue
                raise PointFileError(f"{path}: comment allowed only on line 1")
            parts = line.split(",")
            if cols is None:
                cols = len(parts)
                if cols not in (2, 3):
                    raise PointFileError(f"{path}: expected 2 or 3 columns, found {cols}")
            elif len(parts) != cols:
                raise PointFileError(f"{path}:{lineno}: inconsistent column count")
            try:
                data.append([float(p) for p in parts])
            except ValueError as exc:
                raise PointFileError(f"{path}:{lineno}: {exc}") from None
    if cols is None:
        if header_cols is not None:
            return PointSet.empty(header_cols)
        raise PointFileError(f"{path}: no points found")
    m = np.array(data, dtype=np.float64)
    return PointSet(tuple(m[:, j].copy() for j in range(cols)))


def read_points_device(path, device=None):
    """Format sniffed from the magic (pointfile.py:108-118): PTS1 straight
    to the device, CSV parsed on the host; (n, dim) float64 CUDA tensor."""
    try:
        with open(path, "rb") as fh:
            head = fh.read(4)
    except OSError as exc:
        raise PointFileError(f"{path}: {exc}") from None
    if head == _MAGIC:
        return read_points_binary_device(path, device)
    ps = read_points_csv(path)
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    return torch.from_numpy(ps.as_rows()).to(dev)


UNIFORM_KINDS = {"unit-square": 2, "unit-cube": 3}


def generate_device(kind, n, seed=0, start=0, layout="columns", device=None):
    """Device-side uniform-box cloud, bit-identical to datagen.generate(kind,
    n, seed, start=start): a tuple of dim 1-D CUDA tensors (layout
    "columns") or an (n, dim) tensor ("rows").  Only the uniform kinds are
    generated on the device: the others go through libm functions whose
    device versions differ from the host's in the last bit."""
    if kind not in UNIFORM_KINDS:
        raise ValueError(f"{kind!r} is not generated on the device (libm-based kinds are host-only); "
                         f"device kinds: {sorted(UNIFORM_KINDS)}")
    if n < 0 or start < 0:
        raise ValueError("n and start must be >= 0")
    dim = UNIFORM_KINDS[kind]
    d = torch.cuda.current_device() if device is None else device
    dev = torch.device("cuda", d)
    rows = layout == "rows"
    out = torch.empty((n, dim) if rows else (dim, n), dtype=torch.float64, device=dev)
    with torch.cuda.device(d):
        rc = _lib.lib().sh_uniform_points(_lib.context(d), dim, n, seed & 0xFFFFFFFFFFFFFFFF, start,
                                          1 if rows else 0, out.data_ptr(),
                                          torch.cuda.current_stream(dev).cuda_stream)
    if rc != _lib.SH_OK:
        raise RuntimeError(f"sh_uniform_points failed ({rc}): {_lib.last_error()}")
    return out if rows else tuple(out[c] for c in range(dim))
