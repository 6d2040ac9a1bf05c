"""GPU, full size: the device hull against the REFERENCE itself on the
BASELINE configs it can run (C1, C2, C3, C3', C4-cube), through digests the
reference produced in the build container (tests/golden/make_digests.py,
tests/golden/digests.json): the sorted vertex indices, the vertex rows in
discovery order (byte for byte), the iteration count and the per-round
(live, kept, segments) trace.  The clouds come from the package's generator,
which is bit-identical to the reference's (tests/test_pointio.py)."""

import hashlib
import json
import os

import numpy as np
import pytest
import torch

import paper_1201_2936_b200 as P
from paper_1201_2936_b200.datagen import generate

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

DIGESTS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "digests.json")))
KINDS = {"C1": ("unit-square", 1_000_000), "C2": ("uniform-disk", 100_000_000),
         "C3": ("on-circle", 10_000_000), "C3n": ("near-circle", 10_000_000),
         "C4c": ("unit-cube", 10_000_000)}


@pytest.mark.parametrize("name", [k for k in KINDS if k in DIGESTS])
def test_full_size_matches_reference_digest(name):
    dg = DIGESTS[name]
    kind, n = KINDS[name]
    cols = generate(kind, n, 0)
    assert n == dg["n"]
    d = tuple(torch.from_numpy(c).cuda() for c in cols)
    if len(cols) == 2:
        idx, res = P.hull_indices_2d(d, return_info=True)
    else:
        idx, _, res = P.hull_indices_3d(d, return_info=True)
    tr = P.trace()
    idx = idx.cpu().numpy()
    assert idx.size == dg["h"] and res.iterations == dg["iterations"]
    assert hashlib.sha256(np.sort(idx).astype("<i8").tobytes()).hexdigest() == dg["sorted_idx_sha256"]
    rows = np.column_stack([c[idx] for c in cols])
    assert hashlib.sha256(rows.tobytes()).hexdigest() == dg["rows_sha256"]
    assert tr[:, :3].tolist() == dg["trace"]
