"""Accuracy of the nonbonded kernel's branch-free fp64 math (table exp/log,
MUFU-seeded Halley rsqrt/rcp/rcbrt) against 40-digit mpmath, over the input
ranges the pair evaluation uses."""
import mpmath as mp
import numpy as np
import pytest
import torch

import gen
import paper_1706_07772_b200 as rx

pytestmark = pytest.mark.gpu
mp.mp.dps = 40


def test_device_math_ulps(params):
    rng = np.random.default_rng(3)
    x = np.concatenate([rng.uniform(-40, 40, 4000), rng.uniform(1e-3, 2000, 4000), 10 ** rng.uniform(-3, 3.3, 2000),
                        [1.0, 0.5, 2.0, 64.0, 100.0, 0.81, 1000.0]])
    s = gen.make_config(0)
    ctx = rx.Reax(len(s.pos), s.box, params, gen.CUTOFFS, device=torch.device("cuda:0"))
    out = ctx.selftest_math(torch.from_numpy(x)).cpu().numpy()
    worst = np.zeros(5)
    for i, v in enumerate(x):
        V = mp.mpf(v)
        refs = [mp.exp(V) if abs(v) < 700 else None] + ([mp.log(V), 1 / mp.sqrt(V), 1 / V, V ** (mp.mpf(-1) / 3)] if v > 0 else [None] * 4)
        for c, ref in enumerate(refs):
            if ref is None:
                continue
            if c == 1:
                err = abs(out[i, c] - ref) / max(abs(ref), 1)   # ln: absolute near 1
            else:
                err = abs(out[i, c] - ref) / abs(ref)
            worst[c] = max(worst[c], float(err))
    assert np.all(worst < 5e-16), worst
