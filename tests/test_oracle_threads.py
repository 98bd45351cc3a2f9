"""The oracle is row-parallel (oracle.c header; SURVEY.md §8(c) "std::thread
over atom rows"; "parallel build ... produces identical entries to
serial build").  Every row is computed on its own in a fixed order
and per-row partials are combined in row order, so 1 thread and T threads give
bitwise-identical results.  The row (gather) forms are cross-checked against
the literal forms: Alg. 2's scatter loop over the brute-force half list
(PAPER.md:162-196), the digest of the stored list, the bond list from the
stored half list."""
import numpy as np
import pytest

import gen
import oracle

CUT = gen.CUTOFFS
KEYS = ("hrow", "hcol", "brow", "bcol", "mirror", "raw", "delta", "corr", "E", "F")


@pytest.fixture(scope="module")
def tiny():
    return gen.make_system(700, (21.0, 23.5, 22.0), gen.SEED_BASE + 611)


@pytest.mark.parametrize("T", [2, 3, 8])
def test_one_vs_T_threads_bitwise(c0, params, tiny, T):
    for s in (c0, tiny):
        a = oracle.evaluate(s, params, CUT, threads=1)
        b = oracle.evaluate(s, params, CUT, threads=T)
        for k in KEYS:
            assert np.array_equal(a[k], b[k]), k
        ca, da = oracle.digest_cells(a["pos"], s.box, CUT["r_nonb"], threads=1)
        cb, db = oracle.digest_cells(a["pos"], s.box, CUT["r_nonb"], threads=T)
        assert np.array_equal(ca, cb) and np.array_equal(da, db)
        bp = gen.make_bond_params()
        Ea, Fa = oracle.bond_energy(a["pos"], s.type, s.box, params, bp, a["brow"], a["bcol"], a["raw"], a["delta"],
                                    threads=1)
        Eb, Fb = oracle.bond_energy(a["pos"], s.type, s.box, params, bp, a["brow"], a["bcol"], a["raw"], a["delta"],
                                    threads=T)
        assert Ea == Eb and np.array_equal(Fa, Fb)


def test_rows_match_alg2_scatter(c0, params, tiny):
    """Gather over full rows == Alg. 2's scatter over the brute-force half list
    (same pair function, another summation order: rounding only)."""
    for s in (c0, tiny):
        pos = oracle.wrap(s.pos, s.box)
        hrow, hcol = oracle.half_list(pos, s.box, CUT["r_nonb"], mode="brute")
        Es, Fs = oracle.nonbonded(pos, s.type, s.q, s.box, params, CUT["r_nonb"], hrow, hcol)
        Er, Fr = oracle.nonbonded_rows(pos, s.type, s.q, s.box, params, CUT["r_nonb"])
        assert np.all(np.abs(Er - Es) <= 1e-12 * np.abs(Es)), (Er, Es)
        assert np.max(np.abs(Fr - Fs) / (1 + np.abs(Fs))) <= 1e-11


def test_stream_forms_match_stored_list(c0, params, tiny):
    """The c3/c4 forms (no stored half list) equal the stored-list forms:
    digests of the grid rows == digests of the canonical CSR (exact), bonds
    from the grid at r_bond == bonds from the half list (exact)."""
    for s in (c0, tiny):
        ref = oracle.evaluate(s, params, CUT)
        st = oracle.evaluate_stream(s, params, CUT)
        c, d = oracle.digest(len(s.pos), ref["hrow"], ref["hcol"])
        assert np.array_equal(st["cnt"], c) and np.array_equal(st["dig"], d)
        for k in ("brow", "bcol", "mirror", "raw", "delta", "corr", "E", "F"):
            assert np.array_equal(st[k], ref[k]), k


def test_hbonds_cells_match_definition(c0, params, tiny):
    """O9 H-bond lists from the grid (row-parallel, c3/c4) == the O(N^2)
    definition; 1 vs T threads bitwise."""
    il = oracle.ILIST
    for s in (c0, tiny):
        ref = oracle.evaluate(s, params, CUT)
        a = oracle.hbonds(ref["pos"], s.type, s.box, ref["brow"], il["r_hb"], il["h_type"], il["acc_mask"])
        for T in (1, 5):
            b = oracle.hbonds(ref["pos"], s.type, s.box, ref["brow"], il["r_hb"], il["h_type"], il["acc_mask"],
                              mode="cells", threads=T)
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
