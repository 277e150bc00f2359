"""Pins for the fp64 oracle (runs on CPU, -m "not gpu").

Each test pins the oracle to something other than itself: values printed in
the paper (tests/golden/), closed forms, an independent symbolic expansion
(sympy), point evaluation of the polynomial, finite differences, invariances
and special cases.  Citations are PAPER.md line numbers.
"""
import math
import os

import numpy as np
import pytest

import seeded_inputs as si
from oracle import OracleIndex, adam_update, basis_count, gd_update

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    rows = []
    with open(os.path.join(GOLD, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append([int(t) for t in line.split()])
    return np.array(rows)


# ---------------------------------------------------------------- bases ----

def test_paper_md_example_order():
    """for n=d=2, m_d = (x1^2, x1x2, x2^2) -- in that order."""
    gold = _load("paper_md_n2_d2.txt")
    h = OracleIndex(2, 2)
    assert h.N == 3
    np.testing.assert_array_equal(h.alpha(), gold)


def test_paper_coefficient_counts():
    """PAPER.md:240-256 table and: coefficient / monomial counts."""
    for n, D, count in _load("paper_counts.txt"):
        assert basis_count(int(n), int(D)) == count


@pytest.mark.parametrize("n,d", [(4, 3), (8, 4), (10, 5), (12, 6), (17, 5)])
def test_counts_closed_form(n, d):
    """there are C(k+d-1, k-1) degree-d monomials in k variables."""
    h_count_d = basis_count(n, d)
    assert h_count_d == math.comb(n + d - 1, n - 1)
    assert basis_count(n, 2 * d) == math.comb(n + 2 * d - 1, n - 1)


@pytest.mark.parametrize("n,D", [(3, 2), (4, 3), (5, 4), (3, 6)])
def test_basis_is_bijection_and_prefix_closed(n, D):
    """Every row has degree D, rows are distinct, all C(n+D-1,D) appear, and the
    colex order puts the monomials in the first m variables first (m < n)."""
    h = OracleIndex(n, D)
    A = h.alpha()
    assert A.shape == (math.comb(n + D - 1, D), n)
    assert np.all(A.sum(axis=1) == D)
    assert len({tuple(r) for r in A}) == A.shape[0]
    for m in range(1, n):
        k = math.comb(m + D - 1, D)
        assert np.all(A[:k, m:] == 0)
        np.testing.assert_array_equal(A[:k, :m], OracleIndex(m, D).alpha())


@pytest.mark.parametrize("n,d", [(2, 2), (3, 2), (4, 3), (3, 4)])
def test_pair_ranks_are_products(n, d):
    """rank(alpha_i + alpha_j) indexes the degree-2d basis row alpha_i + alpha_j."""
    h = OracleIndex(n, d)
    A, B = h.alpha(), h.beta()
    P = h.pair_ranks()
    S = A[:, None, :].astype(int) + A[None, :, :].astype(int)
    np.testing.assert_array_equal(B[P.astype(np.int64)], S)
    np.testing.assert_array_equal(P, P.T)


# -------------------------------------------------------------- forward ----

def _poly_coeffs_sympy(A, B, V):
    """Independent brute force: expand sum_k (m_d . v_k)^2 symbolically."""
    sp = pytest.importorskip("sympy")
    n = A.shape[1]
    xs = sp.symbols(f"x0:{n}")

    def mono(e):
        t = sp.Integer(1)
        for v, k in enumerate(e):
            t *= xs[v] ** int(k)
        return t

    ms = [mono(e) for e in A]
    total = 0
    for k in range(V.shape[1]):
        q = sum(sp.Rational(int(V[i, k])) * ms[i] for i in range(len(ms)))
        total += sp.expand(q * q)
    P = sp.Poly(sp.expand(total), *xs)
    out = np.zeros(B.shape[0])
    for t, e in enumerate(B):
        out[t] = float(P.coeff_monomial(mono(e)))
    return out


@pytest.mark.parametrize("n,d,r", [(2, 2, 2), (3, 2, 3), (2, 3, 2), (3, 3, 2)])
def test_forward_matches_symbolic_expansion(n, d, r):
    """PAPER.md:72-76 (Eq. 2): coefficients of sum_k q_k^2 with q_k = m_d . v_k,
    checked against sympy's expansion (integer V, so both sides are exact)."""
    h = OracleIndex(n, d)
    rng = np.random.default_rng(n * 100 + d * 10 + r)
    V = rng.integers(-3, 4, size=(h.N, r)).astype(np.float64)
    got = h.forward(V)
    want = _poly_coeffs_sympy(h.alpha(), h.beta(), V)
    np.testing.assert_array_equal(got, want)


def test_spec_worked_examples():
    """(x1^2+x2^2)^2 = x1^4 + 2x1^2x2^2 + x2^4 and adding (x1x2)^2 gives
    x1^4 + 3x1^2x2^2 + x2^4 (hand expansion)."""
    h = OracleIndex(2, 2)  # m_d = (x1^2, x1x2, x2^2), beta = (x1^4, x1^3x2, ..., x2^4)
    np.testing.assert_array_equal(h.forward(np.array([[1.0], [0.0], [1.0]])), [1, 0, 2, 0, 1])
    V = np.array([[1.0, 0.0], [0.0, 1.0], [1.0, 0.0]])
    np.testing.assert_array_equal(h.forward(V), [1, 0, 3, 0, 1])


@pytest.mark.parametrize("n,d", [(3, 2), (4, 3)])
def test_forward_unit_square(n, d):
    """Closed form: V = e_i (one square, q = x^alpha_i) gives p = x^(2 alpha_i)."""
    h = OracleIndex(n, d)
    A = h.alpha()
    for i in range(h.N):
        V = np.zeros((h.N, 1))
        V[i, 0] = 1.0
        c = h.forward(V)
        k = h.rank2d((2 * A[i]).astype(np.uint8))[0]
        want = np.zeros(h.M)
        want[k] = 1.0
        np.testing.assert_array_equal(c, want)


@pytest.mark.parametrize("n,d,r", [(3, 2, 4), (4, 3, 6), (5, 2, 3)])
def test_forward_point_evaluation(n, d, r):
    """sum_beta coef_beta x^beta == sum_k (m_d(x) . v_k)^2 at random points."""
    h = OracleIndex(n, d)
    V = si.gaussian(h.N, r, 1.0, seed=7, stream=99).astype(np.float64)
    c = h.forward(V)
    X = si.points(50, n, seed=3)
    A, B = h.alpha().astype(np.float64), h.beta().astype(np.float64)
    for x in X:
        md = np.prod(x[None, :] ** A, axis=1)
        mb = np.prod(x[None, :] ** B, axis=1)
        lhs = float(c @ mb)
        rhs = float(np.sum((md @ V) ** 2))
        assert abs(lhs - rhs) <= 1e-10 * max(1.0, abs(rhs))


def test_forward_orthogonal_invariance():
    """coef(V Q) = coef(V) for orthogonal Q: V Q Q^T V^T = V V^T."""
    h = OracleIndex(4, 3)
    V = si.gaussian(h.N, 7, 1.0, seed=1, stream=98).astype(np.float64)
    Q, _ = np.linalg.qr(np.random.default_rng(0).standard_normal((7, 7)))
    np.testing.assert_allclose(h.forward(V @ Q), h.forward(V), rtol=1e-12, atol=1e-12)


def test_coef_sample_matches_forward():
    h = OracleIndex(4, 3)
    V = si.gaussian(h.N, 5, 1.0, seed=2, stream=98).astype(np.float64)
    full = h.forward(V)
    betas = np.arange(0, h.M, 7)
    np.testing.assert_allclose(h.coef_sample(V, betas), full[betas], rtol=1e-13, atol=1e-13)


# ------------------------------------------------------------- gradient ----

@pytest.mark.parametrize("n,d,r", [(3, 2, 4), (2, 3, 3)])
def test_gradient_finite_difference(n, d, r):
    """dL/dV of Eq. 2 against central differences, every coordinate."""
    h = OracleIndex(n, d)
    rng = np.random.default_rng(11)
    V = rng.standard_normal((h.N, r))
    p = rng.standard_normal(h.M)
    loss, g, _, _ = h.loss_grad(V, p)
    eps = 1e-6
    fd = np.zeros_like(V)
    for i in range(h.N):
        for k in range(r):
            Vp = V.copy(); Vp[i, k] += eps
            Vm = V.copy(); Vm[i, k] -= eps
            fd[i, k] = (h.loss_grad(Vp, p, False)[0] - h.loss_grad(Vm, p, False)[0]) / (2 * eps)
    np.testing.assert_allclose(g, fd, rtol=1e-6, atol=1e-6 * np.abs(fd).max())


def test_gradient_is_4RV():
    """dL/dV = 4 R V with R_ij = res[rank(alpha_i+alpha_j)] (explicit matrix)."""
    h = OracleIndex(3, 3)
    rng = np.random.default_rng(5)
    V = rng.standard_normal((h.N, 4))
    p = rng.standard_normal(h.M)
    loss, g, coef, res = h.loss_grad(V, p)
    assert abs(loss - np.sum((coef - p) ** 2)) < 1e-12 * loss
    R = res[h.pair_ranks().astype(np.int64)]
    np.testing.assert_allclose(g, 4 * R @ V, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(h.grad_rows(V, res, [0, 3, h.N - 1]), g[[0, 3, h.N - 1]], rtol=1e-13)


def test_planted_is_stationary():
    """At V = W with p = coef(W W^T) the loss and the gradient vanish."""
    h = OracleIndex(4, 3)
    W = si.planted_w(h.N, 10, seed=0).astype(np.float64)
    p = h.forward(W)
    loss, g, _, _ = h.loss_grad(W, p)
    assert loss == 0.0
    assert np.all(g == 0.0)


# ------------------------------------------------------------ optimisers ----

def test_gd_update_rule():
    V = np.array([1.0, -2.0, 3.0])
    g = np.array([0.5, 0.5, -1.0])
    np.testing.assert_array_equal(gd_update(V, g, 0.1), V - 0.1 * g)


def test_adam_first_step_and_zero_grad():
    """Adam: at t=1 bias correction gives m^=g, v^=g^2, so the
    step is lr*g/(|g|+eps) ~ lr*sign(g); zero gradient leaves V unchanged."""
    V = np.array([1.0, 2.0])
    g = np.array([3.0, -0.25])
    V1, m, v = adam_update(V, g, np.zeros(2), np.zeros(2), 1e-3, 0.9, 0.999, 1e-8, 1)
    np.testing.assert_allclose(V - V1, 1e-3 * np.sign(g), rtol=1e-6)
    V2, _, _ = adam_update(V, np.zeros(2), np.zeros(2), np.zeros(2), 1e-3, 0.9, 0.999, 1e-8, 1)
    np.testing.assert_array_equal(V2, V)


def test_adam_hand_computed_three_steps():
    """Adam (Kingma & Ba, Alg. 1) worked by hand for three steps
    with distinct beta1 = 1/2, beta2 = 3/4, lr = 1, eps = 0 and gradients
    1, 3, -2 (all moments exact binary fractions):
        t=1: m = 1/2,    v = 1/4,        m^ = 1,    v^ = 1      -> step 1
        t=2: m = 7/4,    v = 39/16,      m^ = 7/3,  v^ = 39/7   -> step (7/3)/sqrt(39/7)
        t=3: m = -1/8,   v = 181/64,     m^ = -1/7, v^ = 181/37 -> step (-1/7)/sqrt(181/37)
    A beta1 <-> beta2 swap, a missing bias correction or a bias correction
    with the wrong t changes every step after the first."""
    x, m, v = np.array([5.0]), np.zeros(1), np.zeros(1)
    want_m = [0.5, 7 / 4, -1 / 8]
    want_v = [0.25, 39 / 16, 181 / 64]
    want_x = [5.0 - 1.0]
    want_x.append(want_x[-1] - (7 / 3) / math.sqrt(39 / 7))
    want_x.append(want_x[-1] - (-1 / 7) / math.sqrt(181 / 37))
    for t, g in enumerate([1.0, 3.0, -2.0], start=1):
        x, m, v = adam_update(x, np.array([g]), m, v, 1.0, 0.5, 0.75, 0.0, t)
        assert m[0] == want_m[t - 1] and v[0] == want_v[t - 1]
        assert abs(x[0] - want_x[t - 1]) <= 1e-15 * abs(want_x[t - 1])


def test_adam_matches_torch_optim_adam():
    """The oracle's Adam over 8 steps against an independent implementation,
    torch.optim.Adam on fp64 CPU tensors (foreach/fused off): parameters and
    both moments after every step, non-default betas and eps, gradients that
    change sign and scale from step to step."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(17)
    V = rng.standard_normal((7, 5))
    lr, b1, b2, eps = 3e-2, 0.8, 0.95, 1e-6
    P = torch.tensor(V.copy(), dtype=torch.float64, requires_grad=True)
    opt = torch.optim.Adam([P], lr=lr, betas=(b1, b2), eps=eps, foreach=False, fused=False)
    m, v = np.zeros_like(V), np.zeros_like(V)
    for t in range(1, 9):
        g = rng.standard_normal(V.shape) * (10.0 ** rng.uniform(-3, 2)) * (-1) ** t
        V, m, v = adam_update(V, g, m, v, lr, b1, b2, eps, t)
        P.grad = torch.tensor(g, dtype=torch.float64)
        opt.step()
        st = opt.state[P]
        np.testing.assert_allclose(m, st["exp_avg"].numpy(), rtol=1e-13, atol=0)
        np.testing.assert_allclose(v, st["exp_avg_sq"].numpy(), rtol=1e-13, atol=0)
        np.testing.assert_allclose(V, P.detach().numpy(), rtol=1e-13, atol=1e-15)


def test_adam_scalar_quadratic():
    """100 Adam steps on (x-3)^2 from x=0 with lr=0.1 end within 0.5 of 3."""
    x, m, v = np.zeros(1), np.zeros(1), np.zeros(1)
    for t in range(1, 101):
        x, m, v = adam_update(x, 2 * (x - 3), m, v, 0.1, 0.9, 0.999, 1e-8, t)
    assert abs(x[0] - 3) < 0.5


# ----------------------------------------------- threaded oracle helpers ----

def test_forward_threaded_matches_forward():
    """forward_threaded (row ranges of the same pair loop on host threads) is
    forward() up to fp64 addition order; exact on integer V."""
    h = OracleIndex(4, 3)
    V = si.gaussian(h.N, 9, 1.0, seed=4, stream=98).astype(np.float64)
    np.testing.assert_allclose(h.forward_threaded(V, threads=3), h.forward(V), rtol=1e-13, atol=1e-13)
    Vi = np.random.default_rng(3).integers(-3, 4, size=(h.N, 4)).astype(np.float64)
    np.testing.assert_array_equal(h.forward_threaded(Vi, threads=5), h.forward(Vi))


def test_grad_and_descent_threaded_match_c():
    """grad_rows_threaded == grad_rows; descent_threaded (Python loop over the
    threaded loss/gradient and the oracle's update routines) == or_descent."""
    h = OracleIndex(3, 3)
    rng = np.random.default_rng(8)
    V = rng.standard_normal((h.N, 4)) * 0.3
    p = h.forward(rng.standard_normal((h.N, 2)) * 0.3)
    res = rng.standard_normal(h.M)
    rows = np.arange(h.N)[::-1]
    np.testing.assert_array_equal(h.grad_rows_threaded(V, res, rows, threads=3), h.grad_rows(V, res, rows))
    for kind, lr in (("gd", 1e-2), ("adam", 1e-2)):
        Vc, Lc = h.descent(V, p, kind, 5, lr, b1=0.8, b2=0.9, eps=1e-7)
        Vs, Lt = h.descent_threaded(V, p, kind, 5, lr, b1=0.8, b2=0.9, eps=1e-7, threads=2)
        assert len(Vs) == 6
        np.testing.assert_allclose(Vs[-1], Vc, rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(Lt, Lc, rtol=1e-12)


def test_descent_config0_reaches_1e8():
    """BASELINE config 0 (n=4, 2d=6, r=20, planted r*=10): 2000 GD steps reach a
    relative residual <= 1e-8 (both the Eq. 2 ratio and the norm ratio)."""
    c = si.CONFIGS["c0_n4_2d6"]
    h = OracleIndex(c.n, c.d)
    p = h.forward(si.planted_w(h.N, c.r_star, 0))
    V, L = h.descent(si.v0(h.N, c.r, 0), p, "gd", 2000, 0.02)
    pn = float(p @ p)
    assert L[-1] / pn <= 1e-8
    assert math.sqrt(L[-1] / pn) <= 1e-8


def test_sphere_power_target_term():
    """The eps-term generator of BASELINE config 3: (x1^2+x2^2)^2 has
    coefficients (1, 0, 2, 0, 1) on (x1^4, x1^3x2, ..., x2^4), and in general
    the generated coefficients evaluate to |x|^(2d) at random points."""
    h = OracleIndex(2, 2)
    np.testing.assert_array_equal(si.sphere_power_coefficients(h.beta(), 2), [1, 0, 2, 0, 1])
    h = OracleIndex(4, 3)
    c = si.sphere_power_coefficients(h.beta(), 3)
    B = h.beta().astype(np.float64)
    for x in si.points(5, 4, seed=2):
        assert abs(c @ np.prod(x[None, :] ** B, axis=1) - np.sum(x ** 2) ** 3) < 1e-9 * np.sum(x ** 2) ** 3
