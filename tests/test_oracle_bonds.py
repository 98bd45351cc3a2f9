"""Pins for oracle O3-O5 (BO' terms B1-B2, full bond list, Delta', f1..f5, B8).

Independent pins: closed forms at r = r0 (pow(1,p) = 1), monotonicity,
special cases (Delta' = 0 gives f1 = 1 exactly; huge -p_boc5 gives
f4 = f5 = 1; huge p_boc2 makes f3 a soft minimum), brute-force bond
enumeration, list symmetry/mirror invariants and the
row-sum identity of Delta'.
"""
import numpy as np
import pytest

import gen
import oracle

CUT = gen.CUTOFFS


def test_bo_raw_at_r0_closed_form(params):
    p = params
    for ti, tj in [(0, 0), (0, 3), (1, 2)]:
        r0s = 0.5 * (p.r_sigma[ti] + p.r_sigma[tj])
        r0p = 0.5 * (p.r_pi[ti] + p.r_pi[tj])
        r0pp = 0.5 * (p.r_pipi[ti] + p.r_pipi[tj])
        assert oracle.bo_raw(r0s, ti, tj, p)[0] == np.exp(p.p_bo1[ti, tj])
        assert oracle.bo_raw(r0p, ti, tj, p)[1] == np.exp(p.p_bo3[ti, tj])
        assert oracle.bo_raw(r0pp, ti, tj, p)[2] == np.exp(p.p_bo5[ti, tj])


def test_bo_raw_monotone_and_sum(params):
    rs = np.linspace(0.5, 5.0, 400)
    for ti in range(4):
        for tj in range(4):
            v = np.array([oracle.bo_raw(r, ti, tj, params) for r in rs])
            # strictly decreasing until it underflows (so the r_BOmax prefilter is valid)
            dv = np.diff(v[:, 3])
            assert np.all(dv <= 0) and np.all(dv[v[1:, 3] > 1e-200] < 0)
            assert np.all(v[:, :3] >= 0) and np.all(v[:, :3] <= 1)
            assert np.array_equal(v[:, 3], (v[:, 0] + v[:, 1]) + v[:, 2])
            assert np.array_equal(v, np.array([oracle.bo_raw(r, tj, ti, params) for r in rs]))


def test_bo_raw_pi_switched_off(params):
    p = params.copy()
    p.p_bo3 = np.full((4, 4), -1e5)
    p.p_bo5 = np.full((4, 4), -1e5)
    for r in (1.0, 1.5, 2.0):
        v = oracle.bo_raw(r, 0, 2, p)
        assert v[1] == 0.0 and v[2] == 0.0 and v[3] == v[0]


def _dimer(r, ti, tj, L=25.0):
    pos = np.array([[5.0, 5.0, 5.0], [5.0 + r, 5.0, 5.0]])
    return pos, np.array([ti, tj], np.int32), np.array([L, L, L])


def test_dimer_bond_and_delta(params):
    pos, typ, box = _dimer(1.4, 0, 3)
    hrow, hcol = oracle.half_list(pos, box, 10.0)
    brow, bcol, mir, raw = oracle.bonds(pos, typ, box, params, 5.0, 0.01, hrow, hcol)
    assert brow.tolist() == [0, 1, 2] and bcol.tolist() == [1, 0] and mir.tolist() == [1, 0]
    v = oracle.bo_raw((5.0 + 1.4) - 5.0, 0, 3, params)
    assert np.array_equal(raw[0], v) and np.array_equal(raw[1], v)
    d = oracle.delta(typ, params, brow, raw)
    assert d[0, 0] == v[3] - 4.0 and d[1, 0] == v[3] - 2.0


def test_bond_cut_and_rbond(params):
    # BO' just below the cut: no bond; r beyond r_bond: no bond even if BO' >= cut
    ti, tj = 0, 0
    rs = np.linspace(1.0, 4.0, 3001)
    bo = np.array([oracle.bo_raw(r, ti, tj, params)[3] for r in rs])
    rc = rs[np.argmax(bo < 0.01)]
    for r, expect in ((rc - 0.002, 1), (rc + 0.002, 0)):
        pos, typ, box = _dimer(r, ti, tj)
        hrow, hcol = oracle.half_list(pos, box, 10.0)
        brow, *_ = oracle.bonds(pos, typ, box, params, 5.0, 0.01, hrow, hcol)
        assert brow[-1] == 2 * expect
    pos, typ, box = _dimer(1.2, ti, tj)
    hrow, hcol = oracle.half_list(pos, box, 10.0)
    brow, *_ = oracle.bonds(pos, typ, box, params, 1.1, 0.01, hrow, hcol)
    assert brow[-1] == 0


def test_delta_zero_gives_f1_one(params):
    raw = oracle.bo_raw(1.3, 0, 3, params)
    out, f = oracle.bo_corr_pair(raw, 0.0, 0.0, 0.0, 0.0, 0, 3, params)
    assert f[1] == 2.0 and f[2] == 0.0 and f[0] == 1.0


def test_equal_delta_closed_form(params):
    raw = oracle.bo_raw(1.3, 2, 3, params)
    for d in (-1.5, 0.3, 2.0):
        out, f = oracle.bo_corr_pair(raw, d, d, d, d, 2, 3, params)
        assert abs(f[2] - d) < 4e-15 * max(1, abs(d))               # f3 = d
        assert abs(f[1] - 2 * np.exp(-params.p_boc1 * d)) <= 4e-16 * f[1]
        vi, vj = params.val[2], params.val[3]
        f1 = 0.5 * ((vi + f[1]) / (vi + f[1] + d) + (vj + f[1]) / (vj + f[1] + d))
        assert abs(f[0] - f1) < 1e-14


def test_f3_soft_minimum(params):
    p = params.copy()
    p.p_boc2 = 200.0  # |p Delta| <= 600 stays inside the fp64 exp range
    raw = oracle.bo_raw(1.3, 0, 1, p)
    for di, dj in ((0.5, -0.2), (-1.0, 2.0), (2.0, 2.5)):
        _, f = oracle.bo_corr_pair(raw, di, di, dj, dj, 0, 1, p)
        assert abs(f[2] - (min(di, dj) + np.log(2) / p.p_boc2)) < 1e-12


def test_f4_f5_switched_off(params):
    # Delta'boc = -1000 drives exp(-p_boc3 (p_boc4 BO'^2 - Delta'boc) + p_boc5) below
    # the fp64 underflow threshold, so f4 = f5 = 1 exactly and BO = BO' f1
    raw = oracle.bo_raw(1.2, 0, 3, params)
    out, f = oracle.bo_corr_pair(raw, 0.7, -1000.0, -0.3, -1000.0, 0, 3, params)
    assert f[3] == 1.0 and f[4] == 1.0
    assert out[0] == raw[3] * f[0]
    assert out[2] == raw[1] * f[0] * f[0]


def test_f4_logistic_half_point(params):
    p = params
    raw = oracle.bo_raw(1.25, 1, 2, p)
    pboc3 = np.sqrt(p.b132[1] * p.b132[2])
    pboc4 = np.sqrt(p.b131[1] * p.b131[2])
    pboc5 = np.sqrt(p.b133[1] * p.b133[2])
    dboc = pboc4 * raw[3] ** 2 - pboc5 / pboc3  # makes the exponent zero
    _, f = oracle.bo_corr_pair(raw, dboc, dboc, dboc, dboc, 1, 2, p)
    assert abs(f[3] - 0.5) < 1e-12 and abs(f[4] - 0.5) < 1e-12


def test_corrected_sum(params):
    raw = oracle.bo_raw(1.35, 0, 2, params)
    out, f = oracle.bo_corr_pair(raw, 0.4, 0.4, -0.6, -0.6, 0, 2, params)
    assert abs(out[1] + out[2] + out[3] - out[0]) < 1e-15
    assert abs(out[0] - raw[3] * f[0] * f[3] * f[4]) < 1e-15


def test_bond_list_brute_force_c0(c0, params, c0_oracle):
    o = c0_oracle
    pos = o["pos"]
    rb, cb = oracle.half_list(pos, c0.box, 10.0, "brute")
    want = set()
    for i in range(len(pos)):
        for p_ in range(rb[i], rb[i + 1]):
            j = int(cb[p_])
            d = pos[j] - pos[i]
            d = np.where(d >= 0.5 * c0.box, d - c0.box, np.where(d < -0.5 * c0.box, d + c0.box, d))
            r2 = (d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]
            if r2 <= 25.0 and oracle.bo_raw(np.sqrt(r2), c0.type[i], c0.type[j], params)[3] >= 0.01:
                want.add((i, j))
    brow, bcol = o["brow"], o["bcol"]
    got = {(i, int(bcol[e])) for i in range(len(pos)) for e in range(brow[i], brow[i + 1])}
    assert {(i, j) for (i, j) in got if i < j} == want
    assert got == want | {(j, i) for (i, j) in want}


def test_bond_list_invariants(c0_oracle):
    o = c0_oracle
    brow, bcol, mir, raw, corr = o["brow"], o["bcol"], o["mirror"], o["raw"], o["corr"]
    n = len(brow) - 1
    rowof = np.repeat(np.arange(n), np.diff(brow))
    assert np.array_equal(mir[mir], np.arange(len(bcol)))
    assert np.array_equal(bcol[mir], rowof)
    assert np.array_equal(raw[mir], raw) and np.array_equal(corr[mir], corr)  # bitwise symmetric
    for i in range(n):
        assert np.all(np.diff(bcol[brow[i]:brow[i + 1]]) > 0)
    assert np.all(raw[:, 3] >= 0.01)


def test_delta_row_sum_identity(c0, params, c0_oracle):
    o = c0_oracle
    s = o["delta"][:, 0] + params.val[c0.type]
    assert abs(s.sum() - o["raw"][:, 3].sum()) < 1e-9
    assert np.array_equal(o["delta"][:, 0], o["delta"][:, 1])  # Val_boc = Val in the table (reading 6)


def test_atom_bonds_matches_list(c0, params, c0_oracle):
    o = c0_oracle
    for i in (3, 400, 2000):
        part, raw, dl = oracle.atom_bonds(i, o["pos"], c0.type, c0.box, params, 5.0, 0.01)
        seg = slice(o["brow"][i], o["brow"][i + 1])
        assert part.tolist() == o["bcol"][seg].tolist()
        assert np.array_equal(raw, o["raw"][seg])
        assert np.array_equal(dl, o["delta"][i])


@pytest.mark.parametrize("m", [2.0, 3.0, 0.5])
def test_bo_raw_exponents_closed_form(params, m):
    """B1 at r = r0 * m^(1/p): (r/r0)^p = m, so BO'_k = exp(m * pa_k) for
    each term with its own exponent (sigma: p_bo1, p_bo2; pi: p_bo3, p_bo4;
    pipi: p_bo5, p_bo6).  The three exponents of a pair differ, so a swapped
    or misplaced exponent (or prefactor) fails at m != 1."""
    p = params
    for ti, tj in [(0, 0), (0, 3), (1, 2), (3, 3)]:
        terms = [(p.r_sigma, p.p_bo1, p.p_bo2, 0), (p.r_pi, p.p_bo3, p.p_bo4, 1), (p.r_pipi, p.p_bo5, p.p_bo6, 2)]
        pw = [p.p_bo2[ti, tj], p.p_bo4[ti, tj], p.p_bo6[ti, tj]]
        assert len(set(np.round(pw, 12))) == 3   # distinct exponents: the pin can see a swap
        for r0v, pa, pb, k in terms:
            r0 = 0.5 * (r0v[ti] + r0v[tj])
            r = r0 * m ** (1.0 / pb[ti, tj])
            want = np.exp(m * pa[ti, tj])
            got = oracle.bo_raw(r, ti, tj, p)[k]
            # (r/r0)^p = m to a few ulp; d exp(pa x)/dx relative = |pa| <= 1
            assert abs(got - want) <= 1e-14 * want * max(1.0, m), (ti, tj, k, got, want)
