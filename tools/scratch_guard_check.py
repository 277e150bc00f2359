"""Guard margins around the library's own device allocations (experiment build,
-DSOS_EXPERIMENTS: every cudaMalloc of the library sits between two 64 KB
margins and starts out as 0xFF bytes = NaN).  Runs every call of the ABI on
ragged shapes in every implementation variant, then asks the library which
margins changed (sos_exp_check_guards) and checks that every result is finite
and equals the shipped library's -- a scratch buffer read before it is written,
or read past its end into a float margin, would put a NaN into a result.
python tools/scratch_guard_check.py [quick|big]    (exit code 0 = clean; big = configs 3 and 4 only)
"""
import ctypes, os, subprocess, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import seeded_inputs as si
import paper_2410_19844_b200 as sos
from paper_2410_19844_b200 import build as _b

EXP = "--release" not in sys.argv
if EXP:
    L = sos.load(_b.build(experiments=True))
    L.sos_exp_check_guards.argtypes = [ctypes.POINTER(ctypes.c_int64)]
    L.sos_exp_check_guards.restype = ctypes.c_int

SHAPES = [(5, 3, 37), (7, 3, 85), (7, 4, 163), (9, 4, 321), (9, 4, 700), (11, 4, 1001)]
if "quick" not in sys.argv:
    SHAPES += [(16, 4, 3001)]  # N = 3876: the long-K default plan
if "big" in sys.argv:  # configs 3 and 4 alone, default plan, Adam (what bench.py times)
    SHAPES = [(12, 6, 12376), (17, 5, 20349), (21, 5, 96)]  # the last: N = 53130, segmented-s32 backward
VARIANTS = [dict(), dict(tiny=True), dict(tiny=False, split=True), dict(tiny=False, split=False),
            dict(tiny=False, split=False, narrow_tiles=False, rmax_direct=False),
            dict(tiny=False, split=False, vtq_in_aux=False, vtq_from_update=False, r_headroom=False),
            dict(tiny=False, split=True, tile_w=48)]


def run(n, d, r, opts, kind):
    ix = sos.SosIndex(n, d)
    N, M = ix.N, ix.M
    plan = sos.SosPlan(ix, r, **opts)
    V0 = si.v0(N, r, seed=5)
    W = np.zeros((N, r), np.float32)
    W[:, : max(1, r // 2)] = si.planted_w(N, max(1, r // 2), seed=6)
    V = torch.from_numpy(V0).cuda()
    p = plan.forward(torch.from_numpy(W).cuda())
    res = torch.from_numpy(si.residual_probe(M, seed=7)).cuda()
    out = [plan.forward(V), plan.backward(V, res)]
    loss, grad, rr = plan.loss_grad(V, p, want_res=True)
    out += [loss, grad, rr]
    lr = 1e-3 if kind == "adam" else 0.02 * float(V.norm() / grad.norm())
    plan.opt_init(kind, lr)
    Vd = V.clone()
    out.append(plan.descend(Vd, p, 5).clone())
    out.append(plan.step(Vd, p).clone())
    out.append(Vd)
    Vh = V0.copy()
    plan.opt_init(kind, lr)
    out.append(torch.from_numpy(plan.solve_host(Vh, p.cpu().numpy(), 3)))
    out.append(torch.from_numpy(Vh))
    torch.cuda.synchronize()
    plan.close()
    ix.close()
    return [o.detach().double().cpu().numpy().ravel() for o in out]


N_BIG = "big" in sys.argv


def main():
    results, bad = {}, 0
    for (n, d, r) in SHAPES:
        for vi, opts in enumerate(VARIANTS):
            if n >= 16 and vi not in (0, 2, 4) or N_BIG and vi:
                continue
            for kind in ("adam",) if N_BIG else ("adam", "gd"):
                key = f"{n},{d},{r},{vi},{kind}"
                o = run(n, d, r, opts, kind)
                if not all(np.isfinite(x).all() for x in o):
                    print("NON-FINITE result:", key, [bool(np.isfinite(x).all()) for x in o])
                    bad += 1
                results[key] = np.concatenate([np.atleast_1d(x[:: max(1, x.size // 4096)]) for x in o])
                if EXP:
                    na = ctypes.c_int64()
                    rc = L.sos_exp_check_guards(ctypes.byref(na))
                    if rc != 0:
                        print("GUARD:", key, rc, L.sos_last_error().decode())
                        bad += 1
    return results, bad


def negative_control():
    """The check must see a byte written past an allocation."""
    ix = sos.SosIndex(5, 3)
    plan = sos.SosPlan(ix, 37)
    assert L.sos_exp_check_guards(None) == 0
    assert L.sos_exp_poke_guard() == 0
    seen = L.sos_exp_check_guards(None) < 0
    plan.close()  # frees the poked allocation
    ix.close()
    return seen and L.sos_exp_check_guards(None) == 0


if __name__ == "__main__":
    results, bad = main()
    if EXP and not negative_control():
        print("NEGATIVE CONTROL: a poked margin was not reported")
        bad += 1
    if EXP:  # the same calls through the shipped library, in a fresh process
        path = "/tmp/scratch_guard_release.npz"
        subprocess.run([sys.executable, os.path.abspath(__file__), "--release", "--save=" + path] +
                       [a for a in sys.argv[1:] if a in ("quick", "big")], check=True)
        ref = np.load(path)
        worst = 0.0
        for k, v in results.items():
            e = float(np.linalg.norm(v - ref[k]) / max(np.linalg.norm(ref[k]), 1e-300))
            worst = max(worst, e)
            if not e <= 1e-4:
                print("MISMATCH vs the shipped library:", k, e)
                bad += 1
        print(f"scratch guard check: {len(results)} runs, {bad} problems, worst rel. difference vs the shipped library {worst:.2e}")
    else:
        for a in sys.argv:
            if a.startswith("--save="):
                np.savez(a[7:], **results)
    sys.exit(1 if bad else 0)
