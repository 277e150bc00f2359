"""Streams: every call of the C ABI takes the stream it runs on
(include/sos_b200.h).  A descent on a non-default stream must equal the one on
the default stream, and plans driven from different streams at the same time
-- a long-K plan whose GEMMs pace their K progress over the whole grid (a
bounded wait: DESIGN.md 5.2 "Bounded K-skew"), a split plan with its
cooperative k_mid under programmatic dependent launch, a tiny plan (one
cooperative kernel per call) -- must neither hang nor disturb one another:
each result equals the same plan's run alone.
"""
import numpy as np
import pytest

import seeded_inputs as si

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sos():
    import paper_2410_19844_b200 as m
    m.load()
    return m


class Job:
    def __init__(self, sos, n, d, r, kind, seed, **opts):
        self.ix = sos.SosIndex(n, d)
        N = self.ix.N
        self.plan = sos.SosPlan(self.ix, r, **opts)
        self.V0 = torch.from_numpy(si.v0(N, r, seed=seed)).cuda()
        W = np.zeros((N, r), np.float32)
        W[:, : max(1, r // 2)] = si.planted_w(N, max(1, r // 2), seed=seed + 1)
        self.p = self.plan.forward(torch.from_numpy(W).cuda())
        self.kind = kind
        torch.cuda.synchronize()

    def start(self):
        """Fresh optimiser state and V on the current stream."""
        self.plan.opt_init(self.kind, 1e-3)
        self.V = self.V0.clone()
        self.losses = []

    def descend(self, steps):
        self.losses.append(self.plan.descend(self.V, self.p, steps))

    def result(self):
        return self.V.clone(), torch.cat(self.losses).clone()


def _close(a, b):
    Va, La = a
    Vb, Lb = b
    assert torch.isfinite(Va).all() and torch.isfinite(La).all()
    assert torch.allclose(La, Lb, rtol=1e-5), (La, Lb)
    assert float((Va - Vb).norm() / Vb.norm()) <= 1e-5


@pytest.mark.parametrize("n,d,r,opts", [(4, 3, 20, {}), (9, 4, 700, {}), (9, 4, 700, dict(split=False))])
def test_descend_on_side_stream(sos, n, d, r, opts):
    job = Job(sos, n, d, r, "adam", seed=3, **opts)
    job.start()
    job.descend(5)
    torch.cuda.synchronize()
    want = job.result()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        job.start()
        job.descend(5)
    s.synchronize()
    _close(job.result(), want)


@pytest.mark.timeout(600)
def test_plans_on_concurrent_streams(sos):
    jobs = [
        Job(sos, 16, 4, 3876, "adam", seed=10),            # long K, operands 90 MB: K-skew pacing on
        Job(sos, 9, 4, 700, "adam", seed=20),              # split step (cooperative k_mid, PDL)
        Job(sos, 9, 4, 700, "gd", seed=30, split=False),   # fused step at short K
        Job(sos, 4, 3, 20, "adam", seed=40),               # tiny plan (one cooperative kernel per call)
    ]
    rounds, steps = 3, [4, 7, 5, 50]
    alone = []
    for j, k in zip(jobs, steps):
        j.start()
        for _ in range(rounds):
            j.descend(k)
        torch.cuda.synchronize()
        alone.append(j.result())
    streams = [torch.cuda.Stream() for _ in jobs]
    for s in streams:
        s.wait_stream(torch.cuda.current_stream())
    for j, s in zip(jobs, streams):
        with torch.cuda.stream(s):
            j.start()
    for _ in range(rounds):  # interleaved submissions: the kernels of all four plans contend for the SMs
        for j, s, k in zip(jobs, streams, steps):
            with torch.cuda.stream(s):
                j.descend(k)
    for s in streams:
        s.synchronize()
    for j, want in zip(jobs, alone):
        _close(j.result(), want)


@pytest.mark.timeout(600)
def test_plans_on_host_threads(sos):
    """Distinct plans driven from distinct host threads (ctypes drops the GIL
    inside every call), each on its own stream: the library's shared state (the
    per-kernel occupancy cache, the graph capture of sos_descend in
    thread-local mode) must not mix them up."""
    import threading
    jobs = [Job(sos, 9, 4, 700, "adam", seed=50), Job(sos, 9, 4, 700, "adam", seed=60, split=False),
            Job(sos, 8, 4, 330, "gd", seed=70), Job(sos, 4, 3, 20, "adam", seed=80)]
    alone = []
    for j in jobs:
        j.start()
        for _ in range(4):
            j.descend(5)
        torch.cuda.synchronize()
        alone.append(j.result())
    errors = []

    def run(j):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                j.start()
                for _ in range(4):
                    j.descend(5)
            s.synchronize()
        except Exception as e:  # surfaced below: an exception in a thread would otherwise pass silently
            errors.append(e)

    threads = [threading.Thread(target=run, args=(j,)) for j in jobs]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for j, want in zip(jobs, alone):
        _close(j.result(), want)
