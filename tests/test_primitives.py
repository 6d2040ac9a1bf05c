"""Framework primitives (segmented scans, flag permute, compact, scatter):
the paper's Figure 1 / the reference's worked examples, the reference's own
outputs on seeded inputs (tests/golden/golden_prims.npz), and the GPU ops
against them (bit-exact)."""

import os

import numpy as np
import pytest

from oracle import prims as O

GOLD = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_prims.npz"))
NC = int(GOLD["ncases"][0])
SPECS = [(op, d, m) for op in ("sum", "max", "min") for d in ("forward", "backward")
         for m in ("inclusive", "exclusive")]

# test_primitives.py:21-25 (paper Figure 1) and :164-168 (compact example)
FIG1_F = [2, 0, 1, 1, 1, 2, 2, 1]
FIG1_S = [1, 0, 0, 1, 0, 1, 0, 0]
FIG1_P = [2, 0, 1, 3, 4, 6, 7, 5]
FIG1_S2 = [1, 1, 1, 1, 0, 1, 1, 0]
CP_B = [1, 0, 1, 0, 0, 1]
CP_S = [1, 0, 1, 0, 1, 0]
# test_segments.py:47-55 (S8 = paper Figure 1 heads)
SEG_V = [0, 0, 0, 3, 0, 5, 0, 0]
SEG_S = [1, 0, 0, 1, 0, 1, 0, 0]


@pytest.mark.parametrize("ci", range(NC))
def test_oracle_scans_match_reference(ci):
    s = GOLD[f"s{ci}_heads"]
    for op, d, m in SPECS:
        assert np.array_equal(O.segmented_scan(GOLD[f"s{ci}_vi"], s, op, d, m), GOLD[f"s{ci}_{op}_{d}_{m}_i"])
        if op != "sum":
            got = O.segmented_scan(GOLD[f"s{ci}_vf"], s, op, d, m)
            assert got.tobytes() == GOLD[f"s{ci}_{op}_{d}_{m}_f"].tobytes()


@pytest.mark.parametrize("ci", range(NC))
def test_oracle_permute_compact_match_reference(ci):
    s = GOLD[f"s{ci}_heads"]
    for k in (1, 2, 3):
        p, s2 = O.flag_permute(GOLD[f"s{ci}_fp{k}_f"], s, k)
        assert np.array_equal(p, GOLD[f"s{ci}_fp{k}_p"]) and np.array_equal(s2, GOLD[f"s{ci}_fp{k}_s"])
    p, c, s2 = O.compact(GOLD[f"s{ci}_cp_b"], s)
    assert np.array_equal(p, GOLD[f"s{ci}_cp_p"]) and c == int(GOLD[f"s{ci}_cp_len"][0])
    assert np.array_equal(s2, GOLD[f"s{ci}_cp_s"])


def test_oracle_worked_examples():
    p, s2 = O.flag_permute(FIG1_F, FIG1_S, 3)
    assert p.tolist() == FIG1_P and s2.astype(int).tolist() == FIG1_S2
    p, c, s2 = O.compact(CP_B, CP_S)
    assert p.tolist() == [0, 1, 1, 2, 2, 2] and c == 3 and s2.tolist() == [True, True, True]
    assert O.segmented_scan(SEG_V, SEG_S, "sum").tolist() == [0, 0, 0, 3, 3, 5, 5, 5]


# ---------------------------------------------------------------- GPU ops
@pytest.mark.gpu
def test_gpu_worked_examples():
    import paper_1201_2936_b200.primitives as G
    pm, s2 = G.flag_permute(FIG1_F, FIG1_S, 3)
    assert pm.p.tolist() == FIG1_P and s2.astype(int).tolist() == FIG1_S2 and pm.out_len == 8
    pm, s2 = G.compact(CP_B, CP_S)
    assert pm.p.tolist() == [0, 1, 1, 2, 2, 2] and pm.out_len == 3 and s2.tolist() == [True] * 3
    assert G.segmented_scan(SEG_V, SEG_S, G.ScanSpec("sum")).tolist() == [0, 0, 0, 3, 3, 5, 5, 5]
    # test_segments.py:52-55: backward max
    v = [0, 0, 1, 0, 0, 0, 0, 0]
    assert G.segmented_scan(v, SEG_S, G.ScanSpec("max", "backward")).tolist() == [1, 1, 1, 0, 0, 0, 0, 0]


@pytest.mark.gpu
@pytest.mark.parametrize("ci", range(NC))
def test_gpu_matches_reference_golden(ci):
    import paper_1201_2936_b200.primitives as G
    s = GOLD[f"s{ci}_heads"]
    for op, d, m in SPECS:
        spec = G.ScanSpec(op, d, m)
        assert np.array_equal(G.segmented_scan(GOLD[f"s{ci}_vi"], s, spec), GOLD[f"s{ci}_{op}_{d}_{m}_i"])
        if op != "sum":
            got = G.segmented_scan(GOLD[f"s{ci}_vf"], s, spec)
            assert got.tobytes() == GOLD[f"s{ci}_{op}_{d}_{m}_f"].tobytes()
    for k in (1, 2, 3):
        pm, s2 = G.flag_permute(GOLD[f"s{ci}_fp{k}_f"], s, k)
        assert np.array_equal(pm.p, GOLD[f"s{ci}_fp{k}_p"]) and np.array_equal(s2, GOLD[f"s{ci}_fp{k}_s"])
    pm, s2 = G.compact(GOLD[f"s{ci}_cp_b"], s)
    assert np.array_equal(pm.p, GOLD[f"s{ci}_cp_p"]) and pm.out_len == int(GOLD[f"s{ci}_cp_len"][0])
    assert np.array_equal(s2, GOLD[f"s{ci}_cp_s"])


@pytest.mark.gpu
def test_gpu_large_random_vs_oracle_properties():
    import torch
    import paper_1201_2936_b200.primitives as G
    rng = np.random.default_rng(7)
    n = 3_000_000
    s = rng.random(n) < 0.001
    s[0] = True
    v = rng.integers(-10**12, 10**12, n)
    got = G.segmented_scan(v, s, G.ScanSpec("sum"))
    seg = np.cumsum(s) - 1
    tot = np.zeros(seg[-1] + 1, np.int64)
    np.add.at(tot, seg, v)
    assert np.array_equal(G.reduce_broadcast(np.abs(v), s, "sum"), tot[seg] * 0 + np.bincount(seg, np.abs(v)).astype(np.int64)[seg])
    assert got[-1] == v[np.flatnonzero(s)[-1]:].sum()
    # device tensors in, device tensors out; permute is a within-segment bijection
    f = torch.from_numpy(rng.integers(0, 3, n)).cuda()
    pm, s2 = G.flag_permute(f, torch.from_numpy(s).cuda(), 3)
    assert pm.p.is_cuda and s2.is_cuda
    pp = pm.p.cpu().numpy()
    assert np.array_equal(np.sort(pp), np.arange(n))
    hs = G.head_index_broadcast(s)
    assert np.array_equal(pp >= hs, np.ones(n, bool))
    out = G.scatter(f.cpu().numpy(), G.PermutationMap(pp, n))
    # grouped by state inside every segment
    assert np.array_equal(np.sort(out[:1000]), np.sort(f.cpu().numpy()[pp.argsort()][:1000]))


@pytest.mark.gpu
def test_gpu_contract_errors():
    import paper_1201_2936_b200.primitives as G
    from paper_1201_2936_b200 import ContractViolation
    with pytest.raises(ContractViolation):
        G.segmented_scan([0.5, 1.0], [1, 0], G.ScanSpec("sum"))
    with pytest.raises(ContractViolation):
        G.segmented_scan([1, 2], [0, 1], G.ScanSpec("max"))
    with pytest.raises(ContractViolation):
        G.flag_permute([0, 3], [1, 0], 3)
    with pytest.raises(ContractViolation):
        G.scatter(np.arange(3), G.PermutationMap(np.array([0, 0, 1]), 3))
    with pytest.raises(ContractViolation):
        G.scatter(np.arange(3), G.PermutationMap(np.array([0, 1, 5]), 3))
    assert G.segment_ids([1, 0, 1, 1, 0]).tolist() == [0, 0, 1, 2, 2]
