"""Pins of the oracle's QEq (O11),
against things other than its own code:
  * dense brute force for N <= 200: H assembled by an
    O(N^2) minimum-image enumeration from the separately pinned taper and
    shielded-Coulomb kernel functions, solved by numpy.linalg.solve (library);
    the half-stored SpMV equals the dense product;
  * the constrained minimum: q minimises chi.q + 1/2 q^T H q on sum q = 0
    (the KKT system solved densely);
  * a closed form: no pairs within r_nonb (H diagonal) gives
    q_i = -(chi_i - mu)/eta_i, mu = sum(chi/eta)/sum(1/eta);
  * neutrality, residuals below the tolerance, and warm starts (PAPER.md:206:
    good initial guesses cut the iteration count).
"""
import numpy as np
import pytest

import gen
import oracle

R = 10.0


@pytest.fixture(scope="module")
def qp():
    return gen.make_qeq_params()


def _dense_H(pos, type_, box, params, qp):
    n = len(pos)
    H = np.diag(qp.eta[type_]).astype(float)
    for i in range(n):
        for j in range(i + 1, n):
            d = np.array([oracle.min_image(pos[j, k] - pos[i, k], box[k]) for k in range(3)])
            r2 = (d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]
            if r2 <= R * R:
                r = np.sqrt(r2)
                tap, _ = oracle.taper(r, R)
                k, _ = oracle.coulomb_kernel(r, type_[i], type_[j], params)
                H[i, j] = H[j, i] = params.coulomb_c * tap * k
    return H


@pytest.mark.parametrize("seed", range(4))
def test_dense_brute_force(params, qp, seed):
    rng = np.random.default_rng(70 + seed)
    box = rng.uniform(20.05, 23.0, 3)
    s = gen.make_system(int(rng.integers(20, 200)), box, 7000 + seed)
    pos = oracle.wrap(s.pos, s.box)
    hrow, hcol = oracle.half_list(pos, s.box, R)
    H = _dense_H(pos, s.type, s.box, params, qp)
    hval = oracle.qeq_H(pos, s.type, s.box, params, R, hrow, hcol)
    x = rng.normal(size=len(pos))
    y = oracle.qeq_spmv(qp.eta[s.type], hrow, hcol, hval, x)
    assert np.max(np.abs(y - H @ x)) <= 1e-12 * np.max(np.abs(H @ x))
    q, sv, tv, it = oracle.qeq(pos, s.type, s.box, params, R, hrow, hcol, qp.chi, qp.eta, tol=1e-13)
    s_ref = np.linalg.solve(H, -qp.chi[s.type])
    t_ref = np.linalg.solve(H, -np.ones(len(pos)))
    assert np.max(np.abs(sv - s_ref)) <= 1e-10 * np.max(np.abs(s_ref))
    assert np.max(np.abs(tv - t_ref)) <= 1e-10 * np.max(np.abs(t_ref))
    # the constrained minimum of chi.q + 1/2 q^T H q with sum q = 0 (KKT, dense)
    n = len(pos)
    K = np.zeros((n + 1, n + 1))
    K[:n, :n] = H
    K[:n, n] = K[n, :n] = 1.0
    sol = np.linalg.solve(K, np.r_[-qp.chi[s.type], 0.0])
    assert np.max(np.abs(q - sol[:n])) <= 1e-9 * np.max(np.abs(sol[:n]))
    assert abs(q.sum()) <= 1e-12 * n * np.max(np.abs(q))


def test_isolated_atoms_closed_form(params, qp):
    pos = np.array([[2.0, 2.0, 2.0], [14.0, 2.0, 2.0], [2.0, 14.0, 2.0], [2.0, 2.0, 14.0], [14.0, 14.0, 14.0]])
    typ = np.array([0, 1, 2, 3, 3], np.int32)
    box = np.array([24.0, 24.0, 24.0])     # nearest pairs at 12 A > r_nonb
    hrow, hcol = oracle.half_list(pos, box, R)
    assert len(hcol) == 0
    q, s, t, it = oracle.qeq(pos, typ, box, params, R, hrow, hcol, qp.chi, qp.eta, tol=1e-14)
    chi, eta = qp.chi[typ], qp.eta[typ]
    mu = np.sum(chi / eta) / np.sum(1.0 / eta)
    assert np.allclose(q, -(chi - mu) / eta, rtol=1e-14, atol=1e-15)
    assert np.allclose(s, -chi / eta, rtol=1e-15) and np.allclose(t, -1.0 / eta, rtol=1e-15)


def test_c0_residual_neutrality_and_warm_start(c0, c0_oracle, params, qp):
    ref = c0_oracle
    pos, n = ref["pos"], len(c0.pos)
    q, s, t, it = oracle.qeq(pos, c0.type, c0.box, params, R, ref["hrow"], ref["hcol"], qp.chi, qp.eta,
                             tol=oracle.QEQ_TOL)
    hval = oracle.qeq_H(pos, c0.type, c0.box, params, R, ref["hrow"], ref["hcol"])
    ea = qp.eta[c0.type]
    bs = -qp.chi[c0.type]
    rs = bs - oracle.qeq_spmv(ea, ref["hrow"], ref["hcol"], hval, s)
    rt = -1.0 - oracle.qeq_spmv(ea, ref["hrow"], ref["hcol"], hval, t)
    assert np.linalg.norm(rs) <= oracle.QEQ_TOL * np.linalg.norm(bs)
    assert np.linalg.norm(rt) <= oracle.QEQ_TOL * np.sqrt(n)
    assert abs(q.sum()) <= 1e-12 * n
    assert 5 <= it[0] <= 200 and 5 <= it[1] <= 200
    # warm start from the solution of a slightly perturbed system: fewer iterations
    q2, s2, t2, it2 = oracle.qeq(pos, c0.type, c0.box, params, R, ref["hrow"], ref["hcol"], qp.chi, qp.eta,
                                 tol=oracle.QEQ_TOL, s0=s * (1 + 1e-4), t0=t * (1 + 1e-4))
    assert it2[0] < it[0] and it2[1] < it[1]
    assert np.max(np.abs(q2 - q)) <= 1e-4 * np.max(np.abs(q))
