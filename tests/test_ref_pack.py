"""Pins for the independent NumPy CSR packer (oracle/ref_pack.py): SPEC.md's printed
examples, hand-computed offsets, and the CSR invariants (SURVEY.md P-P1 .. P-P5)."""
import json
import os

import numpy as np

import workloads as wl
from oracle.ref_pack import ref_densify, ref_pack


def test_layout_offset_examples(golden_dir):
    """P-P1: SPEC.md:49-50 layout examples, via a single nonzero at (c, r, s) with R=H, S=W."""
    g = json.load(open(os.path.join(golden_dir, "spec_examples.json")))
    for ex in g["layout_offset"]:
        C, H, W, p = ex["C"], ex["H"], ex["W"], ex["pad"]
        c, y, x = ex["cyx"]
        w = np.zeros((1, C, H + 2 * p, W + 2 * p), np.float32)
        w[0, c, y, x] = 1.0
        P = ref_pack(w, H, W, p, 1)
        assert P["colidx"].tolist() == [ex["offset"]]


def test_layout_additivity():
    """SPEC.md:51 / PAPER.md:290-294: f(c,y+r,x+s) = f(c,y,x) + f(0,r,s)."""
    rng = np.random.default_rng(0)
    for _ in range(50):
        C, H, W, p = (int(v) for v in rng.integers(1, 6, 4))
        Hp, Wp = H + 2 * p, W + 2 * p
        f = lambda c, y, x: (c * Hp + y) * Wp + x
        c = int(rng.integers(0, C)); y = int(rng.integers(0, Hp)); x = int(rng.integers(0, Wp))
        r = int(rng.integers(0, Hp - y)); s = int(rng.integers(0, Wp - x))
        w = np.zeros((1, C, Hp, Wp), np.float32)
        w[0, c, y + r, x + s] = 1.0
        assert ref_pack(w, H, W, p, 1)["colidx"][0] == f(c, y, x) + f(0, r, s)


def test_sparsify_example(golden_dir):
    """P-P2: SPEC.md:60 -> rowptr [0,2,3], values [1,2,3]; colidx derived by hand."""
    ex = json.load(open(os.path.join(golden_dir, "spec_examples.json")))["sparsify"][0]
    w = np.array(ex["weight_2x1x2x2"], np.float32)
    for pad, col in ex["colidx_by_pad"].items():
        P = ref_pack(w, 2, 2, int(pad), 1)
        assert P["rowptr"].tolist() == ex["rowptr"]
        assert P["values"].tolist() == ex["values"]
        assert P["colidx"].tolist() == col


def test_worked_example_csr(golden_dir):
    """P-P3: the worked example's kernel [[1,0],[0,-1]] on a 3x3 input."""
    g = json.load(open(os.path.join(golden_dir, "worked_example_conv.json")))
    w = np.array(g["weight_1x1x2x2"], np.float32)
    for case in g["cases"]:
        P = ref_pack(w, 3, 3, case["pad"], 1)
        for key in ("rowptr", "colidx", "values"):
            assert P[key].tolist() == case["csr"][key]


def test_groups_global_channel(golden_dir):
    """P-P4: with groups, offsets encode the GLOBAL input channel."""
    ex = json.load(open(os.path.join(golden_dir, "spec_examples.json")))["groups"][0]
    P = ref_pack(np.array(ex["weight_2x1x1x1"], np.float32), ex["H"], ex["W"], ex["pad"], ex["groups"])
    assert P["rowptr"].tolist() == ex["rowptr"] and P["colidx"].tolist() == ex["colidx"]


def test_signed_zero_dropped_and_bits_kept():
    w = np.array([[[[0.0, -0.0], [np.float32(1e-38), -3.5]]]], np.float32)
    P = ref_pack(w, 2, 2, 0, 1)
    assert P["values"].view(np.uint32).tolist() == np.array([1e-38, -3.5], np.float32).view(np.uint32).tolist()
    assert P["colidx"].tolist() == [2, 3]


def test_invariants_and_roundtrip():
    """P-P5: rowptr monotone, rowptr[K]=nnz, colidx strictly increasing per row and inside
    the row's group channel range, densify(pack(w)) == w, perm a permutation with
    non-increasing nnz inside each group, ties by ascending k."""
    rng = np.random.default_rng(1)
    for _ in range(200):
        L = wl.random_layer(rng, max_c=12, groups=(1, 2, 3, 4))
        w, _ = wl.random_tensors(rng, L, 1)
        P = ref_pack(w, L.H, L.W, L.pad, L.groups)
        rp, ci = P["rowptr"], P["colidx"]
        assert rp[0] == 0 and rp[-1] == len(ci) == np.count_nonzero(w)
        assert np.all(np.diff(rp) >= 0)
        Hp, Wp = L.H + 2 * L.pad, L.W + 2 * L.pad
        Cg, Kg = L.C // L.groups, L.K // L.groups
        for k in range(L.K):
            row = ci[rp[k]:rp[k + 1]]
            assert np.all(np.diff(row) > 0)
            c = row // (Hp * Wp)
            g = k // Kg
            assert np.all((c >= g * Cg) & (c < (g + 1) * Cg))
        d = ref_densify(rp, ci, P["values"], L.K, L.C, L.R, L.S, L.H, L.W, L.pad, L.groups)
        np.testing.assert_array_equal(d.view(np.uint32), np.where(w == 0, 0, w).view(np.uint32))
        perm = P["perm"]
        assert sorted(perm.tolist()) == list(range(L.K))
        cnt = np.diff(rp)
        for g in range(L.groups):
            pg = perm[g * Kg:(g + 1) * Kg]
            assert np.all(pg // Kg == g)
            c = cnt[pg]
            assert np.all(np.diff(c) <= 0)
            for a, b in zip(pg[:-1], pg[1:]):
                if cnt[a] == cnt[b]:
                    assert a < b


def test_empty_rows_and_all_zero():
    w = np.zeros((3, 2, 3, 3), np.float32)
    w[1, 1, 2, 0] = 2.0
    P = ref_pack(w, 4, 4, 1, 1)
    assert P["rowptr"].tolist() == [0, 0, 1, 1]
    assert P["perm"].tolist() == [1, 0, 2]
    Z = ref_pack(np.zeros((2, 1, 1, 1), np.float32), 1, 1, 0, 1)
    assert Z["rowptr"].tolist() == [0, 0, 0] and len(Z["colidx"]) == 0
