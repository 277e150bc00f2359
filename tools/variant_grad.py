"""Gradient (sos_backward) and one sos_descend step at a fixed shape, saved to
an .npz; used by tests/test_gpu_variants.py to check that implementation
variants selected by environment switches give identical results:
    python tools/variant_grad.py n d r out.npz"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import seeded_inputs as si  # noqa: E402
import paper_2410_19844_b200 as sos  # noqa: E402

n, d, r = (int(x) for x in sys.argv[1:4])
ix = sos.SosIndex(n, d)
plan = sos.SosPlan(ix, r)
V = torch.from_numpy(si.v0(ix.N, r, seed=11)).cuda()
res = torch.from_numpy(si.residual_probe(ix.M, seed=12)).cuda()
g = plan.backward(V, res).cpu().numpy()
W = torch.zeros(ix.N, r, device="cuda")
W[:, : max(1, r // 2)] = torch.from_numpy(si.planted_w(ix.N, max(1, r // 2), 13)).cuda()
p = plan.forward(W)
plan.opt_init("adam", 1e-3)
V2 = V.clone()
losses = plan.descend(V2, p, 3).cpu().numpy()
np.savez(sys.argv[4], grad=g, V3=V2.cpu().numpy(), losses=losses)
