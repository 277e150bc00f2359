#!/usr/bin/env python3
"""Context run for the paper's timing table: random SOS
quartics in n = 10 ... 100 variables solved by Adam descent on one B200
through sos_descend, with the device-side stopping rule at
eps_rel = ||coef - p||^2 / ||p||^2 <= 1e-8 (reading R2).

Prints one JSON line per size and a markdown table with the paper's laptop
seconds beside ours.  The inputs follow the planted-SOS recipe of
seeded_inputs (not the paper's uniform-[-1,1] generator), so the comparison is
context, not a like-for-like benchmark.

  python tools/paper_table.py [--sizes q_n10,q_n100] [--out profiles/r1_paper_table.md]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import seeded_inputs as si  # noqa: E402


def run(sos, torch, cfg, lr, max_steps, chunk, target):
    t0 = time.perf_counter()
    ix = sos.SosIndex(cfg.n, cfg.d)
    W = torch.from_numpy(si.planted_w(ix.N, cfg.r_star, seed=0)).cuda()
    pw = sos.SosPlan(ix, cfg.r_star)
    p = pw.forward(W)
    torch.cuda.synchronize()
    pw.close()
    del W
    pn = float(torch.dot(p.double(), p.double()).item())
    V = torch.from_numpy(si.v0(ix.N, cfg.r, seed=0)).cuda()
    plan = sos.SosPlan(ix, cfg.r)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    plan.opt_init("adam", lr)
    plan.set_stop(target)
    t1 = time.perf_counter()
    steps, reached, hist = 0, None, []
    while steps < max_steps:
        ls = plan.descend(V, p, chunk).cpu().numpy() / pn
        hist.append(ls)
        hit = np.nonzero(ls <= target)[0]
        if hit.size:
            reached = steps + int(hit[0])
            break
        steps += chunk
    t_solve = time.perf_counter() - t1
    loss, _, _ = plan.loss_grad(V, p, want_grad=False)
    plan.close()
    ix.close()
    return {"size": cfg.name, "n": cfg.n, "degree": 2 * cfg.d, "N": ix.N, "M": ix.M, "r": cfg.r,
            "r_star": cfg.r_star, "lr": lr, "steps_to_target": reached, "eps_rel_final": float(loss.item()) / pn,
            "solve_s": round(t_solve, 3), "setup_s": round(t_setup, 3),
            "paper_laptop_s": si.PAPER_QUARTIC_SECONDS[cfg.name]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default=",".join(si.PAPER_QUARTICS))
    ap.add_argument("--lr", type=float, default=1e-3)
    ap.add_argument("--max-steps", type=int, default=5000)
    ap.add_argument("--chunk", type=int, default=100)
    ap.add_argument("--target", type=float, default=1e-8)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    import torch
    import paper_2410_19844_b200 as sos
    rows = []
    for name in args.sizes.split(","):
        r = run(sos, torch, si.PAPER_QUARTICS[name], args.lr, args.max_steps, args.chunk, args.target)
        print(json.dumps(r), flush=True)
        rows.append(r)
    lines = ["| n | coefficients M | N = r | steps to eps_rel <= 1e-8 | B200 solve (s) | paper, i7-6500U laptop (s) |",
             "|---:|---:|---:|---:|---:|---:|"]
    for r in rows:
        lines.append(f"| {r['n']} | {r['M']:,} | {r['N']:,} | {r['steps_to_target']} | {r['solve_s']:.2f} | "
                     f"{r['paper_laptop_s']:,.1f} |")
    table = "\n".join(lines)
    print(table)
    if args.out:
        with open(args.out, "w") as f:
            f.write("# Paper timing table, as context (tools/paper_table.py)\n\n"
                    "Random SOS quartics (2d = 4), full-rank factor r = N, planted r* = N/2 Gaussian target\n"
                    "(seeded_inputs recipe, not the paper's uniform generator), Adam lr "
                    f"{args.lr}, device-side stop at eps_rel <= {args.target}.  Solve time = wall clock of the\n"
                    "descent calls (index/plan setup excluded, as the paper excludes problem setup,\n"
                    "PAPER.md:230).  The paper's column is its own laptop timing (PAPER.md:240-255).\n\n"
                    + table + "\n\n```\n" + "\n".join(json.dumps(r) for r in rows) + "\n```\n")


if __name__ == "__main__":
    main()
