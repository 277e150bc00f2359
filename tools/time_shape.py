"""Device time per descent step for an arbitrary (n, d, r) (planted target, Adam):
python tools/time_shape.py n d r [steps] [--kernels] [split=0|1 rmax_direct=0|1 ...] [lib=PATH]
(key=value arguments are sos_plan_opts fields, for same-box A/B runs)"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import seeded_inputs as si
import paper_2410_19844_b200 as sos
if "--exp" in sys.argv:  # the -DSOS_EXPERIMENTS build (environment switches, probes, traces)
    from paper_2410_19844_b200 import build as _b
    sos.load(_b.build(experiments=True))
for a in sys.argv:  # lib=PATH: an alternative build of the library (same-box A/B)
    if a.startswith("lib="):
        sos.load(a[4:])

for a in sys.argv:  # persist=MB: cudaLimitPersistingL2CacheSize for the run (L2 set-aside experiment)
    if a.startswith("persist="):
        from cuda.bindings import runtime as _rt
        torch.cuda.init()
        print("persist:", _rt.cudaDeviceSetLimit(_rt.cudaLimit.cudaLimitPersistingL2CacheSize, int(a[8:]) << 20),
              _rt.cudaDeviceGetLimit(_rt.cudaLimit.cudaLimitPersistingL2CacheSize))
sys.argv = [a for a in sys.argv if not a.startswith("persist=")]

n, d, r = (int(x) for x in sys.argv[1:4])
steps = int(sys.argv[4]) if len(sys.argv) > 4 and sys.argv[4].isdigit() else 20
opts = {k: (int(v) if k == "tile_w" else bool(int(v))) for k, v in (a.split("=") for a in sys.argv[4:] if "=" in a and not a.startswith("lib="))}
ix = sos.SosIndex(n, d)
plan = sos.SosPlan(ix, r, **opts)
rs = max(1, ix.N // 2)
W = torch.zeros(ix.N, r, device="cuda")
W[:, : min(r, rs)] = torch.from_numpy(si.planted_w(ix.N, min(r, rs), 1)).cuda()
p = plan.forward(W)
V = torch.from_numpy(si.v0(ix.N, r, 0)).cuda()
plan.opt_init("adam", 1e-4)
plan.descend(V, p, 44)  # warm-up: every descent graph of a split plan (16, 4, 1 pairs) gets captured here
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
plan.descend(V, p, steps)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
print(f"n={n} d={d} N={ix.N} r={r} {opts} ms/step={ms:.4f} steps/s={1e3 / ms:.1f}")
if "--kernels" in sys.argv:  # per-kernel split (plain launches with events, a few extra us each)
    plan.timing(True)
    plan.descend(V, p, 10)
    torch.cuda.synchronize()
    plan.timing(False)
    print("  per launch (us):", {k: round(ms / max(1, c) * 1e3, 1) for k, (ms, c) in plan.timing_read().items() if c})
