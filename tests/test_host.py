"""Host-side logic of the drop-in API: containers, validation, exceptions,
input generation, and the rule that the product never touches the oracle."""

import os
import re
import sys

import numpy as np
import pytest

import paper_1201_2936_b200 as P
from paper_1201_2936_b200 import datagen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/pkg/src"


def test_exceptions_mirror_reference_hierarchy():
    for e in (P.ContractViolation, P.EmptyInputError, P.DegenerateInputError):
        assert issubclass(e, ValueError)


def test_pointset_validation():
    with pytest.raises(P.ContractViolation):
        P.PointSet((np.zeros(3),))
    with pytest.raises(P.ContractViolation):
        P.PointSet((np.zeros(3), np.zeros(2)))
    with pytest.raises(P.ContractViolation):
        P.PointSet((np.array([0.0, np.nan]), np.zeros(2)))
    ps = P.PointSet.from_rows([(1, 2), (3, 4)])
    assert ps.n == 2 and ps.dim == 2
    assert ps.as_tuples() == [(1.0, 2.0), (3.0, 4.0)]
    with pytest.raises(P.ContractViolation):
        P.Tolerance(-1.0)


def test_dim_mismatch_and_empty_raise_before_device():
    with pytest.raises(P.ContractViolation):
        P.quickhull_2d(P.PointSet.from_rows([(0, 0, 0)]))
    with pytest.raises(P.ContractViolation):
        P.quickhull_3d(P.PointSet.from_rows([(0, 0)]))
    with pytest.raises(P.EmptyInputError):
        P.quickhull_2d(P.PointSet.empty(2))
    with pytest.raises(P.EmptyInputError):
        P.quickhull_3d(P.PointSet.empty(3))


def test_uniform_stream_chunking_is_exact():
    a = datagen.uniform_stream(5, 1000)
    b = datagen.uniform_stream(5, 1000, chunk=7)
    assert a.tobytes() == b.tobytes()
    c = datagen.uniform_stream(5, 400, start=601)
    assert c.tobytes() == a[600:].tobytes()


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")
def test_datagen_matches_reference_generator():
    sys.path.insert(0, REF)
    import seghull
    for kind in ("uniform-disk", "on-circle", "near-circle", "uniform-ball", "on-sphere",
                 "near-sphere"):
        mine = datagen.generate(kind, 3001, 4)
        ref = seghull.generate(seghull.Distribution(kind, 3001, 4))
        for m, r in zip(mine, ref.coords):
            assert m.tobytes() == r.tobytes(), kind
    u = seghull.datagen._uniform_stream(2, 3000)
    assert datagen.generate("unit-cube", 1000, 2)[1].tobytes() == u.reshape(1000, 3)[:, 1].tobytes()


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1201_2936_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")) or f == "Makefile":
                txt = open(os.path.join(dp, f)).read()
                assert not re.search(r"\boracle\b\s*(import|\.)|import\s+oracle|from\s+oracle|qh_oracle",
                                     txt), f
