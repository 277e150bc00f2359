"""Spread of the r_headroom vs exact Adam comparison (tests/test_gpu_variants.py)
over repeated runs: prints the V_3 and dV relative differences per run.
python tools/hr_adam_probe.py [runs] [lib=PATH]"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import seeded_inputs as si
import paper_2410_19844_b200 as sos
for a in sys.argv:
    if a.startswith("lib="):
        sos.load(a[4:])
runs = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 5
ix = sos.SosIndex(20, 4)
r = 96
for run in range(runs):
    out = []
    for hr in (True, False):
        plan = sos.SosPlan(ix, r, split=False, r_headroom=hr)
        V = torch.from_numpy(si.v0(ix.N, r, seed=31)).cuda()
        W = torch.zeros(ix.N, r, device="cuda")
        W[:, :48] = torch.from_numpy(si.planted_w(ix.N, 48, 32)).cuda()
        p = plan.forward(W)
        plan.opt_init("adam", 1e-3)
        V3 = V.clone()
        losses = plan.descend(V3, p, 5).cpu().numpy()
        out.append((V3.cpu().numpy(), V3.cpu().numpy() - V.cpu().numpy(), losses))
        plan.close()
    a, b = out
    v = np.linalg.norm(a[0] - b[0]) / np.linalg.norm(a[0])
    dv = np.linalg.norm(a[1] - b[1]) / np.linalg.norm(a[1])
    ls = np.max(np.abs(a[2] - b[2]) / np.abs(b[2]))
    print(f"run {run}: V3 rel {v:.3e} (bar 3e-5)  dV rel {dv:.3e} (bar 1e-4)  losses {ls:.2e}")
