"""Guard bands around every user buffer of the C ABI (include/sos_b200.h).

Each buffer a call reads or writes (V, p, res, the coefficient / gradient /
loss outputs) is a window inside a larger device allocation whose margins hold
NaN canaries.  After the call the margins must be bit-identical (no write out
of bounds), and the results must agree with the same call on plain buffers: a
read past the end of V, p or res would pull a NaN into a slice maximum, a Gram
entry or the loss.  Ragged shapes (N and r off every tile, vector and K-block
multiple) in every implementation variant: tiny plan, split step, fused step.
The calls go through the library's ctypes handle so that the outputs the
binding would allocate itself are guarded too.
"""
import ctypes

import numpy as np
import pytest

import seeded_inputs as si

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

MARGIN = 4096  # elements on each side; a multiple of 4 keeps the window 16-byte aligned


@pytest.fixture(scope="module")
def sos():
    import paper_2410_19844_b200 as m
    m.load()
    return m


class Guarded:
    """`numel` elements of `dtype` between two NaN-filled margins."""

    def __init__(self, numel, dtype=torch.float32, fill=None):
        self.buf = torch.full((numel + 2 * MARGIN,), float("nan"), dtype=dtype, device="cuda")
        self.win = self.buf[MARGIN:MARGIN + numel]
        if fill is not None:
            self.win.copy_(torch.as_tensor(fill, dtype=dtype).reshape(-1))
        self.numel = numel
        it = torch.int32 if dtype == torch.float32 else torch.int64
        self.before = self.buf.view(it).clone()

    @property
    def ptr(self):
        return ctypes.c_void_p(self.win.data_ptr())

    def margins_intact(self):
        now = self.buf.view(self.before.dtype)
        lo = torch.equal(now[:MARGIN], self.before[:MARGIN])
        hi = torch.equal(now[MARGIN + self.numel:], self.before[MARGIN + self.numel:])
        return lo and hi

    def unchanged(self):
        return torch.equal(self.buf.view(self.before.dtype), self.before)


VARIANTS = {
    "tiny": dict(tiny=True),
    "split": dict(tiny=False, split=True),
    "fused": dict(tiny=False, split=False),
    "fused_wide": dict(tiny=False, split=False, narrow_tiles=False),
}

# N = 35, 84, 126, 210, 495; r off the 4- / 16- / 64- / 160-element grids
SHAPES = [(5, 3, 37), (7, 3, 85), (6, 4, 131), (7, 4, 163), (9, 4, 321)]


def _check_all(bufs):
    for name, b in bufs.items():
        assert b.margins_intact(), f"write outside {name}"


@pytest.mark.parametrize("variant", ["split", "fused", "fused_wide"])  # a tiny plan changes sos_descend only
@pytest.mark.parametrize("n,d,r", SHAPES)
def test_guard_bands_forward_backward_loss_grad(sos, n, d, r, variant):
    from paper_2410_19844_b200.binding import _check, _stream, load
    L = load()
    ix = sos.SosIndex(n, d)
    N, M = ix.N, ix.M
    plan = sos.SosPlan(ix, r, **VARIANTS[variant])
    ref = sos.SosPlan(ix, r, **VARIANTS[variant])
    V0 = si.v0(N, r, seed=31)
    W = np.zeros((N, r), np.float32)
    W[:, : max(1, r // 2)] = si.planted_w(N, max(1, r // 2), seed=32)
    p0 = ref.forward(torch.from_numpy(W).cuda())
    res0 = si.residual_probe(M, seed=33)

    V = Guarded(N * r, fill=V0)
    p = Guarded(M, fill=p0.cpu())
    res_in = Guarded(M, fill=res0)
    coef = Guarded(M)
    grad = Guarded(N * r)
    res_out = Guarded(M)
    loss = Guarded(1, torch.float64)
    bufs = dict(V=V, p=p, res_in=res_in, coef=coef, grad=grad, res_out=res_out, loss=loss)
    Vp = torch.from_numpy(V0).cuda()

    # forward
    _check(L.sos_forward(plan._h, V.ptr, coef.ptr, _stream()))
    torch.cuda.synchronize()
    _check_all(bufs)
    want = ref.forward(Vp)
    assert torch.isfinite(coef.win).all()
    assert torch.allclose(coef.win, want, rtol=1e-5, atol=1e-6 * float(want.abs().max()))

    # backward (deterministic: bit-identical to the plain-buffer run)
    _check(L.sos_backward(plan._h, V.ptr, res_in.ptr, grad.ptr, _stream()))
    torch.cuda.synchronize()
    _check_all(bufs)
    want = ref.backward(Vp, torch.from_numpy(res0).cuda())
    assert torch.equal(grad.win.view(N, r), want)

    # loss + gradient + residual
    grad.win.fill_(float("nan"))
    _check(L.sos_loss_grad(plan._h, V.ptr, p.ptr, loss.ptr, grad.ptr, res_out.ptr, _stream()))
    torch.cuda.synchronize()
    _check_all(bufs)
    l2, g2, r2 = ref.loss_grad(Vp, p0, want_res=True)
    assert torch.isfinite(grad.win).all() and torch.isfinite(res_out.win).all()
    assert abs(loss.win.item() - l2.item()) <= 1e-5 * abs(l2.item())
    assert torch.allclose(res_out.win, r2, rtol=1e-4, atol=1e-6 * float(r2.abs().max()))
    assert torch.allclose(grad.win.view(N, r), g2, rtol=1e-3, atol=1e-5 * float(g2.abs().max()))
    # inputs are read-only
    assert V.unchanged() and p.unchanged() and res_in.unchanged()
    plan.close()
    ref.close()


def _descend_guarded(sos, n, d, r, opts, kind):
    from paper_2410_19844_b200.binding import _check, _stream, load
    L = load()
    ix = sos.SosIndex(n, d)
    N, M = ix.N, ix.M
    plan = sos.SosPlan(ix, r, **opts)
    ref = sos.SosPlan(ix, r, **opts)
    V0 = si.v0(N, r, seed=41)
    W = np.zeros((N, r), np.float32)
    W[:, : max(1, r // 2)] = si.planted_w(N, max(1, r // 2), seed=42)
    p0 = ref.forward(torch.from_numpy(W).cuda())
    steps = 5  # a plain first step, graph-replayed pairs, a plain tail step

    V = Guarded(N * r, fill=V0)
    p = Guarded(M, fill=p0.cpu())
    losses = Guarded(steps, torch.float64)
    loss1 = Guarded(1, torch.float64)
    bufs = dict(V=V, p=p, losses=losses, loss1=loss1)
    Vp = torch.from_numpy(V0.copy()).cuda()

    lr = 1e-3
    if kind == "gd":  # a 2 % step, whatever the size
        g1 = ref.loss_grad(Vp, p0)[1]
        lr = 0.02 * float(Vp.norm() / g1.norm())
    plan.opt_init(kind, lr)
    ref.opt_init(kind, lr)
    _check(L.sos_descend(plan._h, V.ptr, p.ptr, steps, losses.ptr, _stream()))
    _check(L.sos_step(plan._h, V.ptr, p.ptr, loss1.ptr, _stream()))
    torch.cuda.synchronize()
    _check_all(bufs)
    assert p.unchanged()
    lp = ref.descend(Vp, p0, steps)
    l1 = ref.step(Vp, p0)
    assert torch.isfinite(V.win).all()
    assert torch.allclose(losses.win, lp, rtol=1e-5)
    assert abs(loss1.win.item() - l1.item()) <= 1e-5 * abs(l1.item())
    dv = (V.win.view(N, r) - Vp).norm() / (Vp - torch.from_numpy(V0).cuda()).norm()
    assert float(dv) <= 1e-4, float(dv)
    plan.close()
    ref.close()


@pytest.mark.parametrize("kind", ["gd", "adam"])
@pytest.mark.parametrize("variant", ["tiny", "split", "fused"])
@pytest.mark.parametrize("n,d,r", SHAPES)
def test_guard_bands_step_and_descend(sos, n, d, r, variant, kind):
    _descend_guarded(sos, n, d, r, VARIANTS[variant], kind)


@pytest.mark.parametrize("kind", ["gd", "adam"])
def test_guard_bands_long_k_default_plan(sos, kind):
    """N = 3876 (61 K-blocks): the default plan is the long-K one the bench times
    (update fused into the backward, next-step V / V^T slices from the update,
    headroom R scales, K-skew pacing off / on by operand size); r = 3001 is off
    every tile and vector multiple."""
    _descend_guarded(sos, 16, 4, 3001, {}, kind)


@pytest.mark.timeout(900)
def test_scratch_guards_experiment_build():
    """The library's own allocations (index tables, slices, scales, staging,
    optimiser state): tools/scratch_guard_check.py runs every call on ragged
    shapes in every variant through the -DSOS_EXPERIMENTS build, whose
    allocations sit between 64 KB margins and start as NaN bytes, and fails on
    a changed margin, a non-finite result or a difference from the shipped
    library.  A subprocess: this process has the shipped library loaded."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = subprocess.run([sys.executable, os.path.join(root, "tools", "scratch_guard_check.py")],
                         capture_output=True, text=True, timeout=850)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    assert "0 problems" in res.stdout
