"""A/B check of the R packers: the backward's gradient for a fixed residual must
be bit-identical between SOS_RPACK_SYM=0 and =1 (same slices of R)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import seeded_inputs as si
import paper_2410_19844_b200 as sos

cfg = si.CONFIGS[sys.argv[1]]
ix = sos.SosIndex(cfg.n, cfg.d)
plan = sos.SosPlan(ix, cfg.r)
V = torch.from_numpy(si.v0(ix.N, cfg.r, seed=0)).cuda()
res = torch.from_numpy(si.residual_probe(ix.M, seed=1)).cuda()
g = plan.backward(V, res).cpu().numpy()
np.save(sys.argv[2], g[:: max(1, ix.N // 2000)])
