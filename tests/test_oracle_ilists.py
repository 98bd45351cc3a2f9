"""Pins of the oracle's interaction lists (O9; PAPER.md:
154-158, 198-202): the valence-angle (3-body) list over the full bond list and
the hydrogen-bond list.

  * angles: with both thresholds 0 every other bond of the central atom is an
    angle partner, so an entry of row j has deg(j) - 1 partners (closed form);
    the list is symmetric (k in A(j,i) iff i in A(j,k)); with the default
    thresholds it is the subset of that list whose members pass them (and no
    member of the complement does);
  * H-bonds: the O(N^2) definition equals the list filtered from the pinned
    cell-list half list (an independent route); a 4-atom worked example
    (acceptors at 7.4 A in, 7.6 A out, a bonded donor, a non-acceptor) and an
    H atom without bonds (empty row).
"""
import numpy as np
import pytest

import gen
import oracle

IL = oracle.ILIST


@pytest.fixture(scope="module")
def c0ref():
    p = gen.make_params()
    s = gen.make_config(0)
    return s, p, oracle.evaluate(s, p, gen.CUTOFFS)


def _rows(ref):
    n = len(ref["brow"]) - 1
    return np.repeat(np.arange(n), np.diff(ref["brow"]))


def test_angles_zero_thresholds_closed_form(c0ref):
    s, p, ref = c0ref
    assert np.all(ref["corr"][:, 0] > 0)
    off, k = oracle.angles(ref["brow"], ref["bcol"], ref["corr"], 0.0, 0.0)
    deg = np.diff(ref["brow"])
    row = _rows(ref)
    assert np.array_equal(np.diff(off), deg[row] - 1)
    assert len(k) == int((deg * (deg - 1)).sum())
    # partners of entry e = the other entries of its row, in row order
    for e in range(0, len(row), 97):
        j = row[e]
        others = [ref["bcol"][f] for f in range(ref["brow"][j], ref["brow"][j + 1]) if f != e]
        assert k[off[e]:off[e + 1]].tolist() == others


def _triples(ref, off, k):
    row = _rows(ref)
    return {(int(row[e]), int(ref["bcol"][e]), int(x)) for e in range(len(row)) for x in k[off[e]:off[e + 1]]}


def test_angles_symmetric_and_thresholded_subset(c0ref):
    s, p, ref = c0ref
    off0, k0 = oracle.angles(ref["brow"], ref["bcol"], ref["corr"], 0.0, 0.0)
    off, k = oracle.angles(ref["brow"], ref["bcol"], ref["corr"], IL["thb_cut"], IL["thb_cutsq"])
    t0, t = _triples(ref, off0, k0), _triples(ref, off, k)
    assert t and t < t0
    assert all((j, kk, i) in t for (j, i, kk) in t)          # symmetric in the two bonds
    # BO of the bond (j, x)
    bo = {(int(a), int(b)): ref["corr"][e, 0] for e, (a, b) in enumerate(zip(_rows(ref), ref["bcol"]))}
    for (j, i, kk) in t0:
        be, bf = bo[(j, i)], bo[(j, kk)]
        keep = be > IL["thb_cut"] and bf > IL["thb_cut"] and be * bf > IL["thb_cutsq"]
        assert keep == ((j, i, kk) in t)


def test_hbonds_equal_half_list_route(c0ref):
    s, p, ref = c0ref
    off, z = oracle.hbonds(ref["pos"], s.type, s.box, ref["brow"], IL["r_hb"], IL["h_type"], IL["acc_mask"])
    # independent route: the pinned cell-list half list at r_hb, both directions
    hrow, hcol = oracle.half_list(ref["pos"], s.box, IL["r_hb"])
    n = len(s.pos)
    rows = np.repeat(np.arange(n), np.diff(hrow))
    has_bond = np.diff(ref["brow"]) > 0
    acc = ((IL["acc_mask"] >> s.type) & 1).astype(bool)
    want = [[] for _ in range(n)]
    for a, b in zip(rows, hcol):
        for i, zz in ((a, b), (b, a)):
            if s.type[i] == IL["h_type"] and has_bond[i] and acc[zz]:
                want[i].append(int(zz))
    assert off[-1] == sum(len(w) for w in want) and off[-1] > 0
    for i in range(n):
        assert z[off[i]:off[i + 1]].tolist() == sorted(want[i])


def test_hbonds_worked_example():
    p = gen.make_params()
    # H (type 1) bonded to an O (type 3) 1.0 A away; another O at 7.4 A (in),
    # an N (type 2) at 7.6 A (out), a C (type 0, not an acceptor) at 3 A;
    # a second H far away without bonds
    pos = np.array([[5.0, 5.0, 5.0], [6.0, 5.0, 5.0], [5.0, 12.4, 5.0], [5.0, 5.0, 12.6], [5.0, 2.0, 5.0],
                    [15.0, 15.0, 15.0]])
    typ = np.array([1, 3, 3, 2, 0, 1], np.int32)
    box = np.array([25.0, 25.0, 25.0])
    s = gen.System(pos, typ, np.zeros(len(pos)), box)
    ref = oracle.evaluate(s, p, gen.CUTOFFS)
    rows = _rows(ref)
    assert (0, 1) in set(zip(rows.tolist(), ref["bcol"].tolist()))   # the H-O bond exists
    assert ref["brow"][6] - ref["brow"][5] == 0                      # the far H has none
    off, z = oracle.hbonds(ref["pos"], typ, box, ref["brow"], IL["r_hb"], IL["h_type"], IL["acc_mask"])
    assert z[off[0]:off[1]].tolist() == [1, 2]
    assert off[6] - off[5] == 0 and off[1:5].tolist() == [2, 2, 2, 2]
