"""Seeded random shapes (n, d, r) through the whole path against the fp64 oracle:
index tables bit-exact, forward / backward / loss within the north_star bar, and
one sos_descend step against one sos_step (same iteration)."""
import math

import numpy as np
import pytest

import seeded_inputs as si
from oracle import OracleIndex

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _shapes(count=24, seed=2024):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < count:
        n = int(rng.integers(1, 14))
        d = int(rng.integers(1, 7))
        N = math.comb(n + d - 1, d)
        if N > 2500 or math.comb(n + 2 * d - 1, 2 * d) > 400_000:
            continue
        r = int(rng.integers(1, 700))
        out.append((n, d, r))
    return out


def rel_l2(got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    den = np.linalg.norm(want)
    return np.linalg.norm(got - want) / (den if den > 0 else 1.0)


@pytest.fixture(scope="module")
def sos():
    import paper_2410_19844_b200 as m
    m.load()
    return m


@pytest.mark.parametrize("n,d,r", _shapes())
def test_fuzz_shape(sos, n, d, r):
    o = OracleIndex(n, d)
    ix = sos.SosIndex(n, d)
    assert ix.N == o.N and ix.M == o.M
    assert np.array_equal(ix.alpha().cpu().numpy(), o.alpha())
    plan = sos.SosPlan(ix, r)
    V = si.v0(o.N, r, seed=n * 1000 + d * 100 + r)
    W = si.planted_w(o.N, max(1, r // 2), seed=r)
    p = o.forward(W).astype(np.float32)
    Vd = torch.from_numpy(V).cuda()
    pd = torch.from_numpy(p).cuda()
    assert rel_l2(plan.forward(Vd).cpu().numpy(), o.forward(V)) <= 1e-5
    loss, grad, res = plan.loss_grad(Vd, pd, want_res=True)
    loss_o, grad_o, _, res_o = o.loss_grad(V, p)
    assert abs(loss.item() - loss_o) <= 1e-5 * max(loss_o, 1e-30)
    assert rel_l2(res.cpu().numpy(), res_o) <= 1e-5
    assert rel_l2(grad.cpu().numpy(), grad_o) <= 1e-5
    # one descent step two ways: sos_step and sos_descend
    plan.opt_init("adam", 1e-3)
    Vs = Vd.clone()
    plan.step(Vs, pd)
    plan.opt_init("adam", 1e-3)
    Vq = Vd.clone()
    plan.descend(Vq, pd, 1)
    dv_s = Vs.cpu().numpy() - V
    dv_q = Vq.cpu().numpy() - V
    assert rel_l2(dv_q, dv_s) <= 1e-4


def _variant_shapes(count=14, seed=77):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < count:
        n = int(rng.integers(2, 12))
        d = int(rng.integers(1, 6))
        N = math.comb(n + d - 1, d)
        if N > 1200 or math.comb(n + 2 * d - 1, 2 * d) > 200_000:
            continue
        r = int(rng.integers(1, 600))
        opts = [{"split": True, "tiny": False}, {"split": False, "tiny": False}, {"tiny": True},
                {"split": True, "tile_w": 128, "tiny": False},
                {"split": False, "rmax_direct": True, "vtq_from_update": True, "tiny": False},
                {"split": True, "tile_w": 112, "tiny": False}, {"split": False, "tile_w": 144, "tiny": False},
                ][len(out) % 7]
        out.append((n, d, r, opts))
    return out


@pytest.mark.parametrize("n,d,r,opts", _variant_shapes())
def test_fuzz_descend_variants(sos, n, d, r, opts):
    """Random shapes through sos_descend under each step variant (split step,
    fused step, the one-kernel tiny descent, 128 / 112 / 144-wide tiles, direct R
    maxima + V^T slices from the update):
    3 GD steps against the oracle's GD (V_3 - V_0 element-wise) and its losses."""
    o = OracleIndex(n, d)
    ix = sos.SosIndex(n, d)
    plan = sos.SosPlan(ix, r, **opts)
    V0 = si.v0(o.N, r, seed=n * 100 + r)
    p = o.forward(si.planted_w(o.N, max(1, r // 3), seed=r + 1)).astype(np.float32)
    _, g1, _, _ = o.loss_grad(V0, p)
    lr = 0.02 * np.linalg.norm(V0) / max(np.linalg.norm(g1), 1e-30)
    plan.opt_init("gd", lr)
    Vd = torch.from_numpy(V0.copy()).cuda()
    ld = plan.descend(Vd, torch.from_numpy(p).cuda(), 3).cpu().numpy()
    Vo, Lo = o.descent(V0, p, "gd", 3, lr)
    assert rel_l2(Vd.cpu().numpy() - V0, Vo - V0) <= 1e-5
    assert np.allclose(ld, Lo[:3], rtol=1e-5)
