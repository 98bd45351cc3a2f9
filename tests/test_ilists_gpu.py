"""NEXT-3 parity: reax_interaction_lists (CUDA) against the oracle's O9 on the
same seeded inputs — the 3-body (valence-angle) and H-bond lists must be
identical (integer lists, bit-exact)."""
import numpy as np
import pytest
import torch

import gen
import oracle
from gpu_helpers import CUT, gpu_run

pytestmark = pytest.mark.gpu


def _check(system, params, cut=CUT, **kw):
    ao, ak, ho, hz, ref = oracle.interaction_lists(system, params, cut,
                                                    {("acc_mask" if k == "acceptor_mask" else k): v for k, v in kw.items()})
    ctx, _, _ = gpu_run(system, params, cut)
    g = [t.cpu().numpy() for t in ctx.interaction_lists(**kw)]
    assert np.array_equal(g[0], ao), "angle offsets differ"
    assert np.array_equal(g[1], ak), "angle partners differ"
    assert np.array_equal(g[2], ho), "H-bond offsets differ"
    assert np.array_equal(g[3], hz), "H-bond partners differ"
    return ao, ak, ho, hz


def test_c0(params, c0):
    ao, ak, ho, hz = _check(c0, params)
    assert len(ak) > 1000 and len(hz) > 10000


def test_c1(params):
    _check(gen.make_config(1), params)


@pytest.mark.parametrize("seed", range(3))
def test_tiny_boxes_and_thresholds(params, seed):
    rng = np.random.default_rng(200 + seed)
    box = rng.uniform(20.05, 24.0, 3)
    n = int(rng.integers(20, 400))
    kw = [dict(), dict(thb_cut=0.0, thb_cutsq=0.0), dict(thb_cut=0.05, thb_cutsq=0.01, r_hb=5.0,
                                                          acceptor_mask=0b1111)][seed]
    _check(gen.make_system(n, box, 5000 + seed), params, **kw)


def test_invalid_r_hb(params, c0):
    import paper_1706_07772_b200 as rx
    ctx, _, _ = gpu_run(c0, params)
    with pytest.raises(rx.ReaxError):
        ctx.interaction_lists(r_hb=20.0)   # beyond 2 sub-cell sides
