"""Pins of the oracle's species analysis (O10, SURVEY.md §8(f) NEXT-4;
PAPER.md:217-221 §3.4), against things other than its own code:
  * the molecule partition equals the connected components of scipy's
    csgraph routine (library reference) on random graphs, labelled by their
    smallest atom index and renumbered 1..M in that order;
  * species counts equal a plain Counter over per-molecule compositions;
  * worked examples: two water molecules give the single species H2O x 2
    (SPEC.md:678); a bond order exactly at the threshold (0.3) is not a bond
    ("larger than a threshold"); isolated atoms are molecules;
    per-type-pair thresholds.
"""
from collections import Counter

import numpy as np
import pytest
from scipy.sparse import csr_matrix
from scipy.sparse.csgraph import connected_components

import gen
import oracle


def _graph(n, edges, bo, ntypes=4):
    """Full bond CSR (rows sorted by j) from undirected edges with BO values."""
    rows = {i: [] for i in range(n)}
    for (i, j), b in zip(edges, bo):
        rows[i].append((j, b))
        rows[j].append((i, b))
    brow = [0]
    bcol, corr = [], []
    for i in range(n):
        for j, b in sorted(rows[i]):
            bcol.append(j)
            corr.append([b, b, 0.0, 0.0])
        brow.append(len(bcol))
    return np.array(brow, np.int64), np.array(bcol, np.int32), np.array(corr, np.float64).reshape(-1, 4)


def _expected(n, type_, ntypes, edges, bo, thr):
    keep = [(i, j) for (i, j), b in zip(edges, bo) if b > thr]
    if keep:
        a = np.array(keep)
        A = csr_matrix((np.ones(len(a)), (a[:, 0], a[:, 1])), shape=(n, n))
    else:
        A = csr_matrix((n, n))
    _, lab = connected_components(A, directed=False)
    root = {}
    for i in range(n):
        root.setdefault(lab[i], i)   # smallest index of each component (i ascending)
    order = sorted(root.values())
    rank = {r: k + 1 for k, r in enumerate(order)}
    mol = np.array([rank[root[lab[i]]] for i in range(n)], np.int32)
    comps = Counter()
    for m in range(1, len(order) + 1):
        v = [0] * ntypes
        for i in np.flatnonzero(mol == m):
            v[type_[i]] += 1
        comps[tuple(v)] += 1
    return mol, len(order), comps


@pytest.mark.parametrize("seed", range(12))
def test_random_graphs_match_connected_components(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 400))
    ntypes = int(rng.integers(1, 5))
    type_ = rng.integers(0, ntypes, n).astype(np.int32)
    m = int(rng.integers(0, 2 * n))
    pairs = set()
    for _ in range(m):
        i, j = rng.integers(0, n, 2)
        if i != j:
            pairs.add((min(i, j), max(i, j)))
    edges = sorted(pairs)
    bo = rng.uniform(0.0, 1.0, len(edges))
    brow, bcol, corr = _graph(n, edges, bo)
    mol, M, comp, cnt = oracle.species(type_, ntypes, brow, bcol, corr)
    emol, eM, ecomps = _expected(n, type_, ntypes, edges, bo, 0.3)
    assert M == eM and np.array_equal(mol, emol)
    got = {tuple(c): int(k) for c, k in zip(comp.tolist(), cnt.tolist())}
    assert got == dict(ecomps)
    assert [tuple(c) for c in comp.tolist()] == sorted(got)   # species sorted by composition
    assert cnt.sum() == M


def test_two_waters():
    # O H H O H H (types C=0, H=1, N=2, O=3): O-H bonds 0.95, an H...O contact 0.2
    type_ = np.array([3, 1, 1, 3, 1, 1], np.int32)
    edges = [(0, 1), (0, 2), (3, 4), (3, 5), (2, 3)]
    bo = [0.95, 0.95, 0.95, 0.95, 0.2]
    brow, bcol, corr = _graph(6, edges, bo)
    mol, M, comp, cnt = oracle.species(type_, 4, brow, bcol, corr)
    assert M == 2 and mol.tolist() == [1, 1, 1, 2, 2, 2]
    assert comp.tolist() == [[0, 2, 0, 1]] and cnt.tolist() == [2]


def test_threshold_is_strict_and_per_type_pair():
    type_ = np.array([0, 0, 1, 1], np.int32)
    edges = [(0, 1), (2, 3), (1, 2)]
    bo = [0.3, 0.30000000000000004, 0.5]
    brow, bcol, corr = _graph(4, edges, bo)
    mol, M, _, _ = oracle.species(type_, 2, brow, bcol, corr)
    assert M == 2 and mol.tolist() == [1, 2, 2, 2]     # BO == 0.3 is not a bond
    th = np.array([[0.3, 0.6], [0.6, 0.3]])           # C-H threshold raised above 0.5
    mol, M, comp, cnt = oracle.species(type_, 2, brow, bcol, corr, th)
    assert M == 3 and mol.tolist() == [1, 2, 3, 3]
    assert comp.tolist() == [[0, 2], [1, 0]] and cnt.tolist() == [1, 2]


def test_isolated_atoms_and_empty():
    type_ = np.array([0, 1, 2], np.int32)
    brow, bcol, corr = _graph(3, [], [])
    mol, M, comp, cnt = oracle.species(type_, 3, brow, bcol, corr)
    assert M == 3 and mol.tolist() == [1, 2, 3]
    assert comp.tolist() == [[0, 0, 1], [0, 1, 0], [1, 0, 0]] and cnt.tolist() == [1, 1, 1]
    mol, M, comp, cnt = oracle.species(np.zeros(0, np.int32), 4, np.zeros(1, np.int64), np.zeros(0, np.int32),
                                       np.zeros((0, 4)))
    assert M == 0 and len(comp) == 0


def test_c0_partition(c0, c0_oracle):
    """On c0's corrected bond orders: same partition as the library routine."""
    ref = c0_oracle
    n = len(c0.pos)
    rows = np.repeat(np.arange(n), np.diff(ref["brow"]))
    m = (rows < ref["bcol"])
    edges = list(zip(rows[m].tolist(), ref["bcol"][m].tolist()))
    bo = ref["corr"][m, 0]
    mol, M, comp, cnt = oracle.species(c0.type, 4, ref["brow"], ref["bcol"], ref["corr"])
    emol, eM, ecomps = _expected(n, c0.type, 4, edges, bo, 0.3)
    assert M == eM and np.array_equal(mol, emol)
    assert {tuple(c): int(k) for c, k in zip(comp.tolist(), cnt.tolist())} == dict(ecomps)
