"""Seeded synthetic point clouds for the benchmark configs (host side).

Restates the reference generator (/root/reference/pkg/src/seghull/datagen.py):
splitmix64 stream (datagen.py:53-71) and the six distribution kinds
(datagen.py:99-126), plus the two uniform-box kinds the benchmark configs
name but the reference does not define ("unit square" / "unit cube",
SURVEY.md finding 9): raw splitmix64 uniforms, which are pure integer
arithmetic plus an exact scaling and therefore bit-reproducible on any host.

Output is structure-of-arrays float64, matching ``PointSet``.
"""

import numpy as np

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_MUL1 = np.uint64(0xBF58476D1CE4E5B9)
_MUL2 = np.uint64(0x94D049BB133111EB)
_TO_UNIT = 2.0 ** -53

KINDS_2D = ("uniform-disk", "on-circle", "near-circle", "unit-square")
KINDS_3D = ("uniform-ball", "on-sphere", "near-sphere", "unit-cube")
_DRAWS = {"uniform-disk": 2, "on-circle": 1, "near-circle": 2, "uniform-ball": 5,
          "on-sphere": 4, "near-sphere": 5, "unit-square": 2, "unit-cube": 3}


def _mix(z):
    z = (z ^ (z >> np.uint64(30))) * _MUL1
    z = (z ^ (z >> np.uint64(27))) * _MUL2
    return z ^ (z >> np.uint64(31))


def uniform_stream(seed, count, start=1, chunk=1 << 24):
    """Draws start..start+count-1 of ``seed`` as float64 in [0, 1)
    (datagen.py:67-71; draw k depends only on (seed, k))."""
    out = np.empty(count, dtype=np.float64)
    base = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
    with np.errstate(over="ignore"):
        for lo in range(0, count, chunk):
            hi = min(count, lo + chunk)
            steps = np.arange(start + lo, start + hi, dtype=np.uint64)
            states = base + steps * _GAMMA
            out[lo:hi] = (_mix(states) >> np.uint64(11)).astype(np.float64) * _TO_UNIT
    return out


def _unit_directions(u):
    r1 = np.sqrt(-2.0 * np.log1p(-u[:, 0]))
    r2 = np.sqrt(-2.0 * np.log1p(-u[:, 1]))
    gx = r1 * np.cos(2.0 * np.pi * u[:, 2])
    gy = r1 * np.sin(2.0 * np.pi * u[:, 2])
    gz = r2 * np.cos(2.0 * np.pi * u[:, 3])
    norm = np.sqrt(gx * gx + gy * gy + gz * gz)
    safe = norm > 0
    norm = np.where(safe, norm, 1.0)
    return (np.where(safe, gx / norm, 1.0), np.where(safe, gy / norm, 0.0),
            np.where(safe, gz / norm, 0.0))


def generate(kind, n, seed=0, band=0.01, start=0):
    """SoA tuple of float64 arrays for ``n`` points of ``kind``: points
    start..start+n-1 of the seeded cloud (a shard of a larger cloud)."""
    if kind not in _DRAWS:
        raise ValueError(f"unknown distribution kind {kind!r}")
    dim = 2 if kind in KINDS_2D else 3
    if n == 0:
        return tuple(np.empty(0, np.float64) for _ in range(dim))
    cols = _DRAWS[kind]
    u = uniform_stream(seed, n * cols, start=1 + start * cols).reshape(n, cols)
    if kind in ("unit-square", "unit-cube"):
        return tuple(np.ascontiguousarray(u[:, j]) for j in range(cols))
    if kind == "uniform-disk":
        r, theta = np.sqrt(u[:, 0]), 2.0 * np.pi * u[:, 1]
        return (r * np.cos(theta), r * np.sin(theta))
    if kind == "on-circle":
        theta = 2.0 * np.pi * u[:, 0]
        return (np.cos(theta), np.sin(theta))
    if kind == "near-circle":
        theta = 2.0 * np.pi * u[:, 0]
        r = 1.0 - band * u[:, 1]
        return (r * np.cos(theta), r * np.sin(theta))
    if kind == "uniform-ball":
        r = np.cbrt(u[:, 0])
        dx, dy, dz = _unit_directions(u[:, 1:])
        return (r * dx, r * dy, r * dz)
    if kind == "on-sphere":
        return _unit_directions(u)
    r = 1.0 - band * u[:, 0]
    dx, dy, dz = _unit_directions(u[:, 1:])
    return (r * dx, r * dy, r * dz)
