"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle.

Bars (BASELINE.json north_star): monomial tables and pair ranks bit-exact;
coefficients, loss and gradient within relative L2 error 1e-5 of the oracle;
descent on a planted-SOS target reaches relative residual <= 1e-8.
"""
import math

import numpy as np
import pytest

import seeded_inputs as si
from oracle import OracleIndex
from strata import stratified_rows

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

REL_TOL = 1e-5


def rel_l2(got, want):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    den = np.linalg.norm(want)
    return np.linalg.norm(got - want) / (den if den > 0 else 1.0)


@pytest.fixture(scope="module")
def sos():
    import paper_2410_19844_b200 as m
    m.load()
    return m


_ORACLES = {}


def oracle(n, d):
    if (n, d) not in _ORACLES:
        _ORACLES[(n, d)] = OracleIndex(n, d)
    return _ORACLES[(n, d)]


# (n, d, r): small / ragged / several tiles; includes BASELINE configs 0 and 1
SHAPES = [
    (1, 3, 2),      # univariate: N = 1, M = 1
    (5, 1, 3),      # quadratic forms: N = n
    (2, 2, 1),      # paper example basis, one square
    (4, 3, 20),     # config 0
    (5, 3, 37),     # ragged N = 35, r = 37
    (7, 4, 64),     # N = 210
    (8, 4, 330),    # config 1: N = 330 -> 3 row blocks x 2 col blocks, K ragged
    (9, 4, 300),    # N = 495: 4 x 2 blocks, diagonal straddling tiles
    (3, 9, 33),     # N = 55, high degree
]


@pytest.mark.parametrize("n,d,r", SHAPES)
def test_index_tables_bit_exact(sos, n, d, r):
    o = oracle(n, d)
    ix = sos.SosIndex(n, d)
    assert (ix.N, ix.M) == (o.N, o.M)
    np.testing.assert_array_equal(ix.alpha().cpu().numpy(), o.alpha())
    np.testing.assert_array_equal(ix.beta().cpu().numpy(), o.beta())
    I, J = np.meshgrid(np.arange(o.N), np.arange(o.N), indexing="ij")
    got = ix.pair_ranks(torch.from_numpy(I.ravel()), torch.from_numpy(J.ravel())).cpu().numpy().view(np.uint32)
    np.testing.assert_array_equal(got.reshape(o.N, o.N), o.pair_ranks())


@pytest.mark.parametrize("n,d,r", SHAPES)
def test_forward_parity(sos, n, d, r):
    o = oracle(n, d)
    ix = sos.SosIndex(n, d)
    plan = sos.SosPlan(ix, r)
    V = si.v0(o.N, r, seed=n * 1000 + d * 10 + r)
    coef = plan.forward(torch.from_numpy(V).cuda()).cpu().numpy()
    want = o.forward(V)
    assert rel_l2(coef, want) <= REL_TOL


@pytest.mark.parametrize("n,d,r", SHAPES)
def test_backward_parity(sos, n, d, r):
    o = oracle(n, d)
    ix = sos.SosIndex(n, d)
    plan = sos.SosPlan(ix, r)
    V = si.v0(o.N, r, seed=7 + r)
    res = si.residual_probe(o.M, seed=5 + n)
    g = plan.backward(torch.from_numpy(V).cuda(), torch.from_numpy(res).cuda()).cpu().numpy()
    want = o.grad_rows(V, res, np.arange(o.N))
    assert rel_l2(g, want) <= REL_TOL


@pytest.mark.parametrize("n,d,r", [(4, 3, 20), (8, 4, 330), (9, 4, 300)])
def test_loss_grad_parity_planted(sos, n, d, r):
    o = oracle(n, d)
    ix = sos.SosIndex(n, d)
    plan = sos.SosPlan(ix, r)
    W = si.planted_w(o.N, max(1, r // 2), seed=1)
    V = si.v0(o.N, r, seed=2)
    p = o.forward(W)
    loss_o, g_o, coef_o, res_o = o.loss_grad(V, p)
    loss, g, res = plan.loss_grad(torch.from_numpy(V).cuda(), torch.from_numpy(p.astype(np.float32)).cuda(),
                                  want_res=True)
    # the GPU sees p rounded to fp32; compare against the oracle on that same p
    loss_o, g_o, coef_o, res_o = o.loss_grad(V, p.astype(np.float32))
    assert abs(loss.item() - loss_o) <= REL_TOL * loss_o
    assert rel_l2(res.cpu().numpy(), res_o) <= REL_TOL
    assert rel_l2(g.cpu().numpy(), g_o) <= REL_TOL


@pytest.mark.parametrize("r", [20349, 40000])
def test_forward_long_k_nonnegative(sos, r):
    """Worst case for fp32 accumulation: every product V_ik V_jk >= 0, so every
    partial sum grows monotonically over a long K (r up to 40000)."""
    n, d = 6, 3
    o = oracle(n, d)
    ix = sos.SosIndex(n, d)
    plan = sos.SosPlan(ix, r)
    V = np.abs(si.v0(o.N, r, seed=11))
    coef = plan.forward(torch.from_numpy(V).cuda()).cpu().numpy()
    err = rel_l2(coef, o.forward(V))
    print(f"long-K nonnegative forward rel err {err:.2e}")
    assert err <= REL_TOL
    res = si.residual_probe(o.M, seed=1)
    g = plan.backward(torch.from_numpy(V).cuda(), torch.from_numpy(np.abs(res)).cuda()).cpu().numpy()
    err = rel_l2(g, o.grad_rows(V, np.abs(res), np.arange(o.N)))
    print(f"long-K nonnegative backward rel err {err:.2e}")
    assert err <= REL_TOL


def test_forward_parity_config2(sos):
    """BASELINE config 2 (n=10, 2d=10, N=2002, r=2002): full coefficient vector."""
    c = si.CONFIGS["c2_n10_2d10"]
    o = oracle(c.n, c.d)
    ix = sos.SosIndex(c.n, c.d)
    plan = sos.SosPlan(ix, c.r)
    V = si.v0(o.N, c.r, seed=0)
    coef = plan.forward(torch.from_numpy(V).cuda()).cpu().numpy()
    assert rel_l2(coef, o.forward(V)) <= REL_TOL


def test_adam_and_gd_step_parity(sos):
    n, d, r = 5, 3, 37
    o = oracle(n, d)
    ix = sos.SosIndex(n, d)
    plan = sos.SosPlan(ix, r)
    W = si.planted_w(o.N, 10, seed=3)
    p = o.forward(W).astype(np.float32)
    V0 = si.v0(o.N, r, seed=4)
    for kind, lr in (("gd", 1e-3), ("adam", 1e-3)):
        plan.opt_init(kind, lr)
        Vd = torch.from_numpy(V0.copy()).cuda()
        for _ in range(3):
            plan.step(Vd, torch.from_numpy(p).cuda())
        Vo, _ = o.descent(V0, p, kind, 3, lr)
        # compare the parameter change (the update), relative to its own size
        assert rel_l2(Vd.cpu().numpy() - V0, Vo - V0) <= 1e-4


@pytest.mark.parametrize("kind,lr,steps", [("gd", 0.02, 2000)])
def test_descent_config0_planted(sos, kind, lr, steps):
    """BASELINE config 0: 2000 GD steps from V0 ~ N(0,1/N) on p = coef(W W^T),
    r* = 10.  The final V is checked with the oracle (fp64): relative residual
    ||coef(V) - p||^2 / ||p||^2 <= 1e-8 (reading R2)."""
    c = si.CONFIGS["c0_n4_2d6"]
    o = oracle(c.n, c.d)
    ix = sos.SosIndex(c.n, c.d)
    plan = sos.SosPlan(ix, c.r)
    p = o.forward(si.planted_w(o.N, c.r_star, 0)).astype(np.float32)
    V = torch.from_numpy(si.v0(o.N, c.r, 0)).cuda()
    pd = torch.from_numpy(p).cuda()
    plan.opt_init(kind, lr)
    losses = torch.empty(steps, dtype=torch.float64, device="cuda")
    for t in range(steps):
        plan.step(V, pd, losses[t:t + 1])
    loss_final, _, _, _ = o.loss_grad(V.cpu().numpy(), p, want_grad=False)
    pn = float(np.dot(p.astype(np.float64), p))
    assert loss_final / pn <= 1e-8
    assert losses[-1].item() / pn <= 1e-7


def test_solve_host_matches_device_steps(sos):
    n, d, r = 4, 3, 20
    o = oracle(n, d)
    ix = sos.SosIndex(n, d)
    plan = sos.SosPlan(ix, r)
    p = o.forward(si.planted_w(o.N, 10, 0)).astype(np.float32)
    V0 = si.v0(o.N, r, 0)
    plan.opt_init("gd", 0.02)
    Vh = V0.copy()
    losses = plan.solve_host(Vh, p, 50)
    plan.opt_init("gd", 0.02)
    Vd = torch.from_numpy(V0.copy()).cuda()
    for _ in range(50):
        plan.step(Vd, torch.from_numpy(p).cuda())
    assert rel_l2(Vh, Vd.cpu().numpy()) <= 1e-5
    assert np.all(np.isfinite(losses)) and losses[-1] < losses[0]


@pytest.mark.parametrize("steps", [1, 2, 3, 6])
def test_solve_host_chunked_copy_matches_descend(sos, steps):
    # N = 8855 rows -> 5 row chunks of V shipped by the copy stream during the
    # last step's backward; steps 1..3 cover the graph / plain-step boundaries
    n, d, r = 20, 4, 96
    ix = sos.SosIndex(n, d)
    plan = sos.SosPlan(ix, r)
    V0 = si.v0(ix.N, r, seed=3)
    W = np.zeros((ix.N, r), np.float32)
    W[:, :48] = si.planted_w(ix.N, 48, 4)  # zero columns leave coef(W W^T) unchanged
    Wd = torch.from_numpy(W).cuda()
    p = plan.forward(Wd).cpu().numpy()
    plan.opt_init("adam", 1e-3)
    Vh = V0.copy()
    lh = plan.solve_host(Vh, p, steps)
    plan.opt_init("adam", 1e-3)
    Vd = torch.from_numpy(V0.copy()).cuda()
    ld = plan.descend(Vd, torch.from_numpy(p).cuda(), steps).cpu().numpy()
    assert not np.array_equal(Vh, V0)
    assert rel_l2(Vh, Vd.cpu().numpy()) <= 1e-6
    assert np.allclose(lh, ld, rtol=1e-5)


def test_solve_host_stopped_releases_copy(sos):
    # stopping rule already met: the update never runs, the copy stream must
    # still be released (no hang) and V comes back unchanged
    n, d, r = 20, 4, 96
    ix = sos.SosIndex(n, d)
    plan = sos.SosPlan(ix, r)
    V0 = si.v0(ix.N, r, seed=5)
    p = plan.forward(torch.from_numpy(V0).cuda()).cpu().numpy() * 1.001
    plan.opt_init("adam", 1e-3)
    plan.set_stop(1e-2)
    Vh = V0.copy()
    losses = plan.solve_host(Vh, p, 4)
    assert np.array_equal(Vh, V0)
    assert np.all(np.isfinite(losses))


# ---------------------------------------------------------------- full size --

@pytest.fixture(scope="module", params=["c3_n12_2d12", si.BENCH_CONFIG])
def big(sos, request):
    """BASELINE configs 3 (1.35M coefficients) and 4 (5.3M coefficients)."""
    c = si.CONFIGS[request.param]
    ix = sos.SosIndex(c.n, c.d)
    plan = sos.SosPlan(ix, c.r)
    V = si.v0(ix.N, c.r, seed=0)
    yield c, ix, plan, V
    plan.close()
    ix.close()


def test_full_size_index_sampled(sos, big):
    c, ix, plan, V = big
    o = oracle(c.n, c.d)
    np.testing.assert_array_equal(ix.alpha().cpu().numpy(), o.alpha())
    np.testing.assert_array_equal(ix.beta().cpu().numpy(), o.beta())
    rows = np.array([0, 1, 777, o.N // 2, o.N - 1], dtype=np.int64)
    I = np.repeat(rows, o.N)
    J = np.tile(np.arange(o.N, dtype=np.int64), rows.size)
    got = ix.pair_ranks(torch.from_numpy(I), torch.from_numpy(J)).cpu().numpy().view(np.uint32)
    np.testing.assert_array_equal(got.reshape(rows.size, o.N), o.pair_ranks(rows))


def test_full_size_forward_sampled(sos, big):
    """Sampled coefficients vs the oracle -- random ones, and the squares
    x^(2 alpha_i) and neighbours x^(alpha_i + alpha_(i+1)) of the stratified
    rows, which take their diagonal (weight-1) and near-diagonal entries from
    the forward's diagonal tiles -- plus the point-evaluation identity
    sum_beta coef_beta x^beta = sum_k (m_d(x) . v_k)^2 on the whole vector."""
    c, ix, plan, V = big
    o = oracle(c.n, c.d)
    coef = plan.forward(torch.from_numpy(V).cuda()).cpu().numpy().astype(np.float64)
    rng = np.random.default_rng(0)
    A = o.alpha()
    rows = stratified_rows(o.N)
    nxt = np.minimum(rows + 1, o.N - 1)
    diag = o.rank2d((A[rows].astype(np.int64) * 2).astype(np.uint8))
    near = o.rank2d((A[rows].astype(np.int64) + A[nxt]).astype(np.uint8))
    betas = np.unique(np.concatenate([np.arange(8), rng.integers(0, o.M, 56), [o.M - 1], diag, near]))
    want = o.coef_sample(V, betas)
    err = rel_l2(coef[betas], want)
    print(f"{c.name} forward sampled ({betas.size} coefficients) rel err {err:.2e}")
    assert err <= REL_TOL
    B = o.beta().astype(np.float64)
    Vd = V.astype(np.float64)
    for x in si.points(2, c.n, seed=1) * 0.5:
        lhs = coef @ np.prod(x[None, :] ** B, axis=1)
        rhs = np.sum((np.prod(x[None, :] ** A.astype(np.float64), axis=1) @ Vd) ** 2)
        assert abs(lhs - rhs) <= REL_TOL * abs(rhs)


@pytest.mark.parametrize("nonneg", [False, True])
def test_full_size_backward_sampled(sos, big, nonneg):
    """Backward at full size (K = N): >= 64 stratified rows of 4RV (both CTAs
    of the pair tiles, all lane quarters, first / last / interior row blocks,
    every column tile) vs the oracle's gradient rows, computed on host threads;
    nonneg=True makes every product R_ij V_jk >= 0 (monotone partial sums)."""
    c, ix, plan, V = big
    o = oracle(c.n, c.d)
    res = si.residual_probe(o.M, seed=9)
    if nonneg:
        res, V = np.abs(res), np.abs(V)
    g = plan.backward(torch.from_numpy(V).cuda(), torch.from_numpy(res).cuda())
    rows = stratified_rows(o.N)
    got = g[torch.from_numpy(rows).cuda()].cpu().numpy()
    want = o.grad_rows_threaded(V.astype(np.float64), res, rows)
    err = rel_l2(got, want)
    worst = max(rel_l2(got[k], want[k]) for k in range(rows.size))
    print(f"{c.name} backward (nonneg={nonneg}) {rows.size} rows: rel err {err:.2e}, worst row {worst:.2e}")
    assert err <= REL_TOL
    assert worst <= 4 * REL_TOL


def test_full_size_descend_step_sampled(sos, big):
    """One sos_descend step (the launch configuration bench.py times: forward,
    residual, R slices, backward with the fused update) at full size, on >= 64
    stratified rows against the oracle.  p = coef(V0) - res0 makes the residual
    a known probe, so the oracle needs only gradient rows g.  Three updates:
      * GD, V1 - V0 = -lr g                        (gradient magnitudes, bar 1e-5)
      * Adam with eps = rms(g): V1 - V0 = -lr g / (|g| + eps)   (smooth in g, bar 1e-5)
      * Adam with eps = 1e-8 (bench.py's): ~ -lr sign(g)         (bar 1e-4: entries
        whose g is within the forward's rounding of 0 may take either sign)."""
    c, ix, plan, V = big
    o = oracle(c.n, c.d)
    Vd = torch.from_numpy(V).cuda()
    coef = plan.forward(Vd).cpu().numpy().astype(np.float64)
    res0 = si.residual_probe(o.M, seed=21)
    p = (coef - res0).astype(np.float32)
    # the GPU's residual coef - p is res0 up to the fp32 rounding of p (~1e-7 relative);
    # the oracle gets the seeded res0 itself (no oracle input comes from the CUDA path)
    res_eff = res0.astype(np.float64)
    rows = stratified_rows(o.N)
    g = o.grad_rows_threaded(V.astype(np.float64), res_eff, rows)
    grms = float(np.sqrt(np.mean(g * g)))
    vrms = float(np.sqrt(np.mean(V[rows].astype(np.float64) ** 2)))
    cases = [("gd", 0.05 * vrms / grms, None, 1e-5), ("adam", 1e-3, grms, 1e-5), ("adam", 1e-3, 1e-8, 1e-4)]
    for kind, lr, eps, tol in cases:
        if kind == "gd":
            plan.opt_init("gd", lr)
            want = -lr * g
        else:
            plan.opt_init("adam", lr, eps=eps)
            want = -lr * g / (np.abs(g) + eps)
        V1 = Vd.clone()
        plan.descend(V1, torch.from_numpy(p).cuda(), 1)
        got = V1[torch.from_numpy(rows).cuda()].cpu().numpy().astype(np.float64) - V[rows]
        err = rel_l2(got, want)
        print(f"{c.name} descend step {kind} eps={eps} lr={lr:.3g}: {rows.size} rows rel err {err:.2e}")
        assert err <= tol
    # the host-buffer entry point (bench.py's e2e leg, V shipped back in chunks)
    # agrees; Adam's first step is ~lr sign(g), so the few entries whose g is
    # within the forward's rounding of 0 may flip between runs (atomics order)
    lr = 1e-3
    plan.opt_init("adam", lr)
    V1 = Vd.clone()
    plan.descend(V1, torch.from_numpy(p).cuda(), 1)
    plan.opt_init("adam", lr)
    Vh = V.copy()
    plan.solve_host(Vh, p, 1)
    d = np.abs((Vh - V) - (V1.cpu().numpy() - V))
    assert np.count_nonzero(d > 0.1 * lr) <= 1e-5 * d.size
    assert np.median(d) <= 1e-6 * lr


def test_config3_target_with_eps_term(sos):
    """Config 3's target p = coef(W W^T) + eps (sum x_i^2)^6: the eps term is
    added on the exponent table the index exports; check it on sampled
    coefficients against the oracle (eps = 1e-3)."""
    c = si.CONFIGS["c3_n12_2d12"]
    o = oracle(c.n, c.d)
    ix = sos.SosIndex(c.n, c.d)
    plan_w = sos.SosPlan(ix, c.r_star)
    W = si.planted_w(o.N, c.r_star, seed=0)
    sphere = si.sphere_power_coefficients(ix.beta().cpu().numpy(), c.d)
    p = plan_w.forward(torch.from_numpy(W).cuda()).cpu().numpy().astype(np.float64) + c.eps * sphere
    betas = np.concatenate([np.arange(6), np.random.default_rng(1).integers(0, o.M, 40)])
    want = o.coef_sample(W, betas) + c.eps * si.sphere_power_coefficients(o.beta()[betas], c.d)
    assert rel_l2(p[betas], want) <= REL_TOL


def test_forward_parity_config2b_r4004(sos):
    """BASELINE config 2, over-parameterised r = 4004: sampled coefficients and rows."""
    c = si.CONFIGS["c2b_n10_2d10_r4004"]
    o = oracle(c.n, c.d)
    ix = sos.SosIndex(c.n, c.d)
    plan = sos.SosPlan(ix, c.r)
    V = si.v0(o.N, c.r, seed=3)
    coef = plan.forward(torch.from_numpy(V).cuda()).cpu().numpy()
    betas = np.arange(0, o.M, 97)
    assert rel_l2(coef[betas], o.coef_sample(V, betas)) <= REL_TOL
    res = si.residual_probe(o.M, seed=4)
    g = plan.backward(torch.from_numpy(V).cuda(), torch.from_numpy(res).cuda()).cpu().numpy()
    rows = np.array([0, 1000, o.N - 1])
    assert rel_l2(g[rows], o.grad_rows(V, res, rows)) <= REL_TOL


def test_descent_config1_planted(sos):
    """BASELINE config 1 (n=8, 2d=8, N=330, r=330, planted r*=165): GD on the
    GPU reaches relative residual <= 1e-8 (checked in fp64 by the oracle)."""
    c = si.CONFIGS["c1_n8_2d8"]
    o = oracle(c.n, c.d)
    ix = sos.SosIndex(c.n, c.d)
    plan = sos.SosPlan(ix, c.r)
    p = o.forward(si.planted_w(o.N, c.r_star, 0)).astype(np.float32)
    V = torch.from_numpy(si.v0(o.N, c.r, 0)).cuda()
    pd = torch.from_numpy(p).cuda()
    plan.opt_init("gd", 0.01)
    loss = torch.empty(1, dtype=torch.float64, device="cuda")
    for t in range(4000):
        plan.step(V, pd, loss)
    pn = float(np.dot(p.astype(np.float64), p))
    loss_final, _, _, _ = o.loss_grad(V.cpu().numpy(), p, want_grad=False)
    print(f"config1 descent: gpu {loss.item() / pn:.3e} oracle {loss_final / pn:.3e}")
    assert loss_final / pn <= 1e-8


def test_stop_rule_freezes_v(sos):
    """sos_opt_set_stop: once ||coef - p||^2 <= tol ||p||^2 the step leaves V
    (and the optimiser state) untouched; before that V moves."""
    c = si.CONFIGS["c0_n4_2d6"]
    o = oracle(c.n, c.d)
    ix = sos.SosIndex(c.n, c.d)
    plan = sos.SosPlan(ix, c.r)
    p = o.forward(si.planted_w(o.N, c.r_star, 0)).astype(np.float32)
    pd = torch.from_numpy(p).cuda()
    pn = float(np.dot(p.astype(np.float64), p))
    V = torch.from_numpy(si.v0(o.N, c.r, 0)).cuda()
    plan.opt_init("adam", 1e-2)
    plan.set_stop(1e-6)
    loss = torch.empty(1, dtype=torch.float64, device="cuda")
    for t in range(3000):
        before = V.clone()
        plan.step(V, pd, loss)
        if loss.item() <= 1e-6 * pn:
            break
        assert not torch.equal(before, V)
    assert loss.item() <= 1e-6 * pn
    frozen = V.clone()
    for _ in range(5):
        plan.step(V, pd, loss)
    assert torch.equal(frozen, V)
    lo, _, _, _ = o.loss_grad(V.cpu().numpy(), p, want_grad=False)
    assert lo / pn <= 1.01e-6


@pytest.mark.parametrize("cfg_name,lr", [("c2_n10_2d10", 1e-3), ("c2b_n10_2d10_r4004", 1e-3)])
def test_descent_config2_adam_reaches_1e8(sos, cfg_name, lr):
    """BASELINE config 2 (N=2002, r in {2002, 4004}, planted r*=1001): Adam
     on the GPU reaches eps_rel <= 1e-8; the final V is
    re-checked by the fp64 oracle's full forward."""
    c = si.CONFIGS[cfg_name]
    o = oracle(c.n, c.d)
    ix = sos.SosIndex(c.n, c.d)
    plan = sos.SosPlan(ix, c.r)
    p = o.forward(si.planted_w(o.N, c.r_star, 0)).astype(np.float32)
    pd = torch.from_numpy(p).cuda()
    pn = float(np.dot(p.astype(np.float64), p))
    V = torch.from_numpy(si.v0(o.N, c.r, 0)).cuda()
    plan.opt_init("adam", lr)
    plan.set_stop(0.5e-8)
    losses = torch.empty(2000, dtype=torch.float64, device="cuda")
    for t in range(2000):
        plan.step(V, pd, losses[t:t + 1])
    hist = losses.cpu().numpy() / pn
    reached = int(np.argmax(hist <= 0.5e-8)) if np.any(hist <= 0.5e-8) else None
    lo, _, _, _ = o.loss_grad(V.cpu().numpy(), p, want_grad=False)
    print(f"{cfg_name}: reached 0.5e-8 at step {reached}; oracle eps_rel of final V {lo / pn:.3e}")
    assert reached is not None
    assert lo / pn <= 1e-8


@pytest.mark.parametrize("cfg_name,lr", [("c3_n12_2d12", 5e-4), (si.BENCH_CONFIG, 1e-3)])
def test_descent_full_size_adam_reaches_1e8(sos, cfg_name, lr):
    """BASELINE configs 3 (1.35M coefficients, target + eps (sum x^2)^6) and 4
    (5.3M coefficients): Adam through sos_descend, with the device-side stopping
    rule at eps_rel <= 0.5e-8, reaches the target (device loss, fp64-accumulated).
    The forward at the final V is re-checked against the oracle on sampled
    coefficients, so the loss it reports is the oracle's up to the forward's
    relative error."""
    c = si.CONFIGS[cfg_name]
    ix = sos.SosIndex(c.n, c.d)
    W = torch.from_numpy(si.planted_w(ix.N, c.r_star, 0)).cuda()
    plan_w = sos.SosPlan(ix, c.r_star)
    p = plan_w.forward(W)
    torch.cuda.synchronize()
    plan_w.close()
    del W
    if c.eps:
        sphere = si.sphere_power_coefficients(ix.beta().cpu().numpy(), c.d)
        p = (p.double() + c.eps * torch.from_numpy(sphere).cuda()).float()
    pn = float(torch.dot(p.double(), p.double()).item())
    V = torch.from_numpy(si.v0(ix.N, c.r, 0)).cuda()
    plan = sos.SosPlan(ix, c.r)
    plan.opt_init("adam", lr)
    plan.set_stop(0.5e-8)
    hist = []
    for _ in range(10):
        hist.append(plan.descend(V, p, 100).cpu().numpy() / pn)
        if hist[-1].min() <= 0.5e-8:
            break
    hist = np.concatenate(hist)
    assert np.any(hist <= 0.5e-8), f"min eps_rel {hist.min():.3e} after {hist.size} steps"
    print(f"{cfg_name}: eps_rel <= 0.5e-8 at step {int(np.argmax(hist <= 0.5e-8))}")
    o = oracle(c.n, c.d)
    coef = plan.forward(V).cpu().numpy()
    betas = np.concatenate([np.arange(4), np.random.default_rng(2).integers(0, o.M, 28)])
    Vh = V.cpu().numpy()
    assert rel_l2(coef[betas], o.coef_sample(Vh, betas)) <= REL_TOL
    loss, _, _ = plan.loss_grad(V, p, want_grad=False)
    assert loss.item() / pn <= 1e-8
    plan.close()
    ix.close()


# ------------------------------------------------- slice-arithmetic edge cases --

def test_backward_spiky_residual(sos):
    """Per-row slice scales: one residual 1e6 x larger than the rest (the
    x1^{2d} coefficient, reached by one pair only) must not wash out the other
    entries of the rows that do not contain it, nor those that do."""
    n, d, r = 6, 3, 64
    o = oracle(n, d)
    ix = sos.SosIndex(n, d)
    plan = sos.SosPlan(ix, r)
    V = si.v0(o.N, r, seed=21)
    res = si.residual_probe(o.M, seed=22)
    res[0] *= 1e6
    res[o.M - 1] *= 1e6
    g = plan.backward(torch.from_numpy(V).cuda(), torch.from_numpy(res).cuda()).cpu().numpy()
    want = o.grad_rows(V, res, np.arange(o.N))
    assert rel_l2(g, want) <= REL_TOL
    # rows whose R row holds no spike keep their own relative accuracy
    rows = np.nonzero(np.abs(want).max(axis=1) < 1e3 * np.median(np.abs(want)))[0]
    assert rows.size > 0
    assert rel_l2(g[rows], want[rows]) <= REL_TOL


def test_forward_wide_dynamic_range(sos):
    """Rows and columns of V spanning 12 orders of magnitude: every row (and
    column) is sliced against its own maximum."""
    n, d, r = 5, 3, 48
    o = oracle(n, d)
    ix = sos.SosIndex(n, d)
    plan = sos.SosPlan(ix, r)
    V = si.v0(o.N, r, seed=31).astype(np.float64)
    V *= np.logspace(-6, 6, o.N)[:, None]
    V *= np.logspace(3, -3, r)[None, :]
    V = V.astype(np.float32)
    coef = plan.forward(torch.from_numpy(V).cuda()).cpu().numpy()
    assert rel_l2(coef, o.forward(V)) <= REL_TOL
    res = si.residual_probe(o.M, seed=32)
    g = plan.backward(torch.from_numpy(V).cuda(), torch.from_numpy(res).cuda()).cpu().numpy()
    want = o.grad_rows(V, res, np.arange(o.N))
    assert rel_l2(g, want) <= REL_TOL


def test_forward_segmented_s32_accumulation(sos):
    """K = r = 50000 > 43648: exact s32 accumulation would overflow its bound,
    so the GEMM drains TMEM per segment into fp32 sums; all products >= 0."""
    n, d, r = 6, 3, 50000
    o = oracle(n, d)
    ix = sos.SosIndex(n, d)
    plan = sos.SosPlan(ix, r)
    V = np.abs(si.v0(o.N, r, seed=41))
    coef = plan.forward(torch.from_numpy(V).cuda()).cpu().numpy()
    assert rel_l2(coef, o.forward(V)) <= REL_TOL


def test_zero_rows_and_columns(sos):
    """All-zero rows/columns of V and an all-zero residual: scale 0, exact zeros out."""
    n, d, r = 4, 3, 40
    o = oracle(n, d)
    ix = sos.SosIndex(n, d)
    plan = sos.SosPlan(ix, r)
    V = si.v0(o.N, r, seed=51)
    V[3] = 0.0
    V[:, 7] = 0.0
    coef = plan.forward(torch.from_numpy(V).cuda()).cpu().numpy()
    assert rel_l2(coef, o.forward(V)) <= REL_TOL
    g = plan.backward(torch.from_numpy(V).cuda(), torch.zeros(o.M, device="cuda")).cpu().numpy()
    assert np.all(g == 0.0)
    g0 = plan.backward(torch.zeros_like(torch.from_numpy(V)).cuda(),
                       torch.from_numpy(si.residual_probe(o.M, seed=52)).cuda()).cpu().numpy()
    assert np.all(g0 == 0.0)


# -------------------------------------------------------------- sos_descend --

@pytest.mark.parametrize("variant", ["split", "fused_vtq_update"])
@pytest.mark.parametrize("kind,lr,r", [("adam", 1e-3, 330), ("gd", 5e-3, 330), ("adam", 1e-3, 336)])
def test_descend_matches_steps(sos, kind, lr, r, variant):
    """sos_descend (slices of V_{t+1} written by the update of step t) follows
    the same iteration as repeated sos_step calls, to the slice precision.
    Row 5 and column 9 of V0 are zero, so their first update leaves the
    headroom window of the fused variant and is re-sliced by the fixup kernels
    (VQ row, VTQ row).  r = 336 (a multiple of 4) and r = 330 (rows not 16-byte
    aligned).  "fused_vtq_update": the update in the backward's epilogue warps
    also writes the next step's V^T slices (the default only for long K);
    "split": forward, k_mid, backward storing the gradient, row-block update
    with exact next-step scales (the default for short K)."""
    opts = {"split": True} if variant == "split" else {"split": False, "vtq_from_update": True}
    c = si.CONFIGS["c1_n8_2d8"]
    o = oracle(c.n, c.d)
    ix = sos.SosIndex(c.n, c.d)
    plan = sos.SosPlan(ix, r, **opts)
    p = torch.from_numpy(o.forward(si.planted_w(o.N, c.r_star, 0)).astype(np.float32)).cuda()
    V0 = si.v0(o.N, r, 0)
    V0[5] = 0.0
    V0[:, 9] = 0.0
    steps = 30
    plan.opt_init(kind, lr)
    Vs = torch.from_numpy(V0.copy()).cuda()
    ls = torch.empty(steps, dtype=torch.float64, device="cuda")
    for t in range(steps):
        plan.step(Vs, p, ls[t:t + 1])
    plan.opt_init(kind, lr)
    Vd = torch.from_numpy(V0.copy()).cuda()
    ld = plan.descend(Vd, p, steps)
    torch.cuda.synchronize()
    dv_s = Vs.cpu().numpy() - V0
    dv_d = Vd.cpu().numpy() - V0
    assert rel_l2(dv_d, dv_s) <= 1e-4
    assert np.allclose(ld.cpu().numpy(), ls.cpu().numpy(), rtol=1e-4)
    # and the final V's loss, by the oracle, matches the device loss curve's trend
    lo, _, _, _ = o.loss_grad(Vd.cpu().numpy(), p.cpu().numpy(), want_grad=False)
    assert lo < ld[0].item()


@pytest.mark.parametrize("kind,lr", [("gd", 5e-3), ("adam", 1e-3)])
@pytest.mark.parametrize("steps", [9, 47, 100])
def test_descend_split_graph_cascade_vs_oracle(sos, steps, kind, lr):
    """A split plan's sos_descend replays graphs of 16, 4 and 1 pairs of steps
    (47 = 1 plain + 32 + 8 + 3 x 2; 100 = 1 + 3 x 32 + 2 + 1 plain; 9 = 1 + 8):
    V_t and every loss against the oracle's descent at config 1."""
    c = si.CONFIGS["c1_n8_2d8"]
    o = oracle(c.n, c.d)
    ix = sos.SosIndex(c.n, c.d)
    plan = sos.SosPlan(ix, c.r, split=True, tiny=False)
    p = o.forward(si.planted_w(o.N, c.r_star, 0)).astype(np.float32)
    V0 = si.v0(o.N, c.r, 3)
    plan.opt_init(kind, lr)
    Vd = torch.from_numpy(V0.copy()).cuda()
    ld = plan.descend(Vd, torch.from_numpy(p).cuda(), steps).cpu().numpy()
    Vo, Lo = o.descent(V0, p, kind, steps, lr)
    # loss bar along a trajectory: 1e-4.  The 1e-5 bar holds for L at a given V (tested
    # above); here V_t itself carries the accumulated ~2e-6 and the residual shrinks, so
    # the relative loss error grows with t (GD: ~5e-6 at step 9, 1.2e-5 .. 1.9e-5 at step
    # 100, varying with the order of the forward's atomics; Adam ~7e-7)
    L = Lo[:steps]
    err, lerr = rel_l2(Vd.cpu().numpy() - V0, Vo - V0), np.max(np.abs(ld - L) / L)
    print(f"graph cascade {kind} {steps} steps: dV rel err {err:.2e}, worst loss rel err {lerr:.2e}")
    assert err <= 1e-4
    assert lerr <= 1e-4


def test_descend_reaches_1e8_config2_and_stops(sos):
    """Config 2 through sos_descend with the device-side stopping rule: the
    iteration freezes at the first V with eps_rel <= 0.5e-8, checked by the
    fp64 oracle."""
    c = si.CONFIGS["c2_n10_2d10"]
    o = oracle(c.n, c.d)
    ix = sos.SosIndex(c.n, c.d)
    plan = sos.SosPlan(ix, c.r)
    pf = o.forward(si.planted_w(o.N, c.r_star, 0)).astype(np.float32)
    p = torch.from_numpy(pf).cuda()
    pn = float(np.dot(pf.astype(np.float64), pf))
    V = torch.from_numpy(si.v0(o.N, c.r, 0)).cuda()
    plan.opt_init("adam", 1e-3)
    plan.set_stop(0.5e-8)
    losses = plan.descend(V, p, 600).cpu().numpy() / pn
    hit = np.nonzero(losses <= 0.5e-8)[0]
    assert hit.size > 0
    # frozen after the stop (the loss repeats up to the order of the forward's
    # fp32 atomic reductions), and V does not move in further calls
    assert np.allclose(losses[hit[0]:], losses[hit[0]], rtol=1e-4)
    frozen = V.clone()
    plan.descend(V, p, 5)
    assert torch.equal(frozen, V)
    lo, _, _, _ = o.loss_grad(V.cpu().numpy(), pf, want_grad=False)
    print(f"descend config2: stop at step {hit[0]}, oracle eps_rel {lo / pn:.3e}")
    assert lo / pn <= 1e-8


def test_large_n_sampled(sos):
    """Beyond the BASELINE sizes: n=20, 2d=10 (N = 42,504 monomials, M =
    20,030,010 coefficients, r = N; R rows of 171 KB still take the fused R
    packer, K = 42,752 stays below the exact-s32 segment bound).  Sampled
    coefficients and gradient rows against the oracle, and the
    point-evaluation identity on the full coefficient vector."""
    n, d = 20, 5
    o = oracle(n, d)
    ix = sos.SosIndex(n, d)
    assert (ix.N, ix.M) == (o.N, o.M) == (42504, 20030010)
    r = ix.N
    plan = sos.SosPlan(ix, r)
    V = si.v0(ix.N, r, seed=5)
    Vd = torch.from_numpy(V).cuda()
    coef = plan.forward(Vd).cpu().numpy().astype(np.float64)
    rng = np.random.default_rng(7)
    betas = np.concatenate([[0, 1, o.M - 1], rng.integers(0, o.M, 20)])
    assert rel_l2(coef[betas], o.coef_sample(V, betas)) <= REL_TOL
    res = si.residual_probe(o.M, seed=8)
    g = plan.backward(Vd, torch.from_numpy(res).cuda())
    rows = np.array([3, o.N - 2], dtype=np.int64)
    got = g[torch.from_numpy(rows).cuda()].cpu().numpy()
    assert rel_l2(got, o.grad_rows(V, res, rows)) <= REL_TOL
    x = si.points(1, n, seed=9)[0] * 0.5
    B = o.beta().astype(np.float64)
    lhs = coef @ np.prod(x[None, :] ** B, axis=1)
    A = o.alpha().astype(np.float64)
    rhs = np.sum((np.prod(x[None, :] ** A, axis=1) @ V.astype(np.float64)) ** 2)
    assert abs(lhs - rhs) <= REL_TOL * abs(rhs)
    plan.close()
    ix.close()


# tile-boundary shapes: N just above 160 (B-tile width) and 256 (pair tile
# height), r around the 64-wide K-block and the 160-wide column block
BOUNDARY = [
    (9, 3, 63), (9, 3, 64), (9, 3, 65),          # N = 165
    (11, 3, 159), (11, 3, 160), (11, 3, 161),    # N = 286
    (4, 8, 255), (4, 8, 256), (4, 8, 257),       # N = 165, high degree
    (7, 4, 1), (7, 4, 321),                      # N = 210
]


@pytest.mark.parametrize("n,d,r", BOUNDARY)
def test_boundary_shapes_forward_backward(sos, n, d, r):
    o = oracle(n, d)
    ix = sos.SosIndex(n, d)
    plan = sos.SosPlan(ix, r)
    V = si.v0(o.N, r, seed=100 + r)
    Vd = torch.from_numpy(V).cuda()
    assert rel_l2(plan.forward(Vd).cpu().numpy(), o.forward(V)) <= REL_TOL
    res = si.residual_probe(o.M, seed=200 + r)
    g = plan.backward(Vd, torch.from_numpy(res).cuda()).cpu().numpy()
    assert rel_l2(g, o.grad_rows(V, res, np.arange(o.N))) <= REL_TOL


@pytest.mark.parametrize("variant", ["split", "fused"])
@pytest.mark.parametrize("n,d,r", [(2, 2, 1), (7, 4, 1), (5, 3, 3), (1, 3, 2), (4, 3, 20)])
def test_descend_tiny_shapes_vs_oracle(sos, n, d, r, variant):
    """Degenerate sizes through sos_descend (r = 1: one square; N = 1: a
    univariate form; rows shorter than a float4): 3 GD steps against the
    oracle's GD, and the losses."""
    o = oracle(n, d)
    ix = sos.SosIndex(n, d)
    plan = sos.SosPlan(ix, r, split=(variant == "split"))
    W = si.planted_w(o.N, max(1, r // 2), seed=8)
    p = o.forward(W).astype(np.float32)
    V0 = si.v0(o.N, r, seed=9)
    lr = 1e-2
    plan.opt_init("gd", lr)
    Vd = torch.from_numpy(V0.copy()).cuda()
    ld = plan.descend(Vd, torch.from_numpy(p).cuda(), 3).cpu().numpy()
    Vo, Lo = o.descent(V0, p, "gd", 3, lr)
    assert rel_l2(Vd.cpu().numpy() - V0, Vo - V0) <= 1e-5
    assert np.allclose(ld, Lo[:3], rtol=1e-5)


def test_forward_full_vector_config3(sos):
    """BASELINE config 3 (N = r = 12376): the WHOLE coefficient vector (M =
    1,352,078) against the oracle's pair loop, run on all host threads (~1 min
    on the 16-core B200 host); relative L2 and the worst relative error over
    the coefficients whose magnitude is at least the vector's rms."""
    c = si.CONFIGS["c3_n12_2d12"]
    o = oracle(c.n, c.d)
    ix = sos.SosIndex(c.n, c.d)
    plan = sos.SosPlan(ix, c.r)
    V = si.v0(o.N, c.r, seed=3)
    coef = plan.forward(torch.from_numpy(V).cuda()).cpu().numpy().astype(np.float64)
    want = o.forward_threaded(V)
    err = rel_l2(coef, want)
    big = np.abs(want) >= np.sqrt(np.mean(want ** 2))
    worst = float(np.max(np.abs(coef[big] - want[big]) / np.abs(want[big])))
    print(f"config 3 full forward: rel L2 {err:.2e}, worst relative error on |coef| >= rms {worst:.2e}")
    assert err <= REL_TOL
    assert worst <= 1e-4
    plan.close()
    ix.close()


def test_backward_full_config2(sos):
    """BASELINE config 2 (N = r = 2002): every row of 4RV against the oracle
    (host threads), through the split plan's backward (128-wide column tiles)."""
    c = si.CONFIGS["c2_n10_2d10"]
    o = oracle(c.n, c.d)
    ix = sos.SosIndex(c.n, c.d)
    plan = sos.SosPlan(ix, c.r)
    V = si.v0(o.N, c.r, seed=4)
    res = si.residual_probe(o.M, seed=6)
    g = plan.backward(torch.from_numpy(V).cuda(), torch.from_numpy(res).cuda()).cpu().numpy()
    want = o.grad_rows_threaded(V.astype(np.float64), res, np.arange(o.N))
    err = rel_l2(g, want)
    print(f"config 2 full backward: rel L2 {err:.2e}")
    assert err <= REL_TOL
    plan.close()
    ix.close()
