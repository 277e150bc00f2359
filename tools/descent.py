#!/usr/bin/env python3
"""Full descent on a planted-SOS target, on the GPU, through the C ABI.

BASELINE.json north_star: "a descent run on a planted-SOS target must reach
relative residual <= 1e-8".  This driver runs sos_step (GD or Adam,
PAPER.md:221) on one BASELINE.json config until the relative residual
eps_rel = ||coef(V V^T) - p||^2 / ||p||^2 (reading R2) reaches the
target, optionally with a step-size schedule, and prints one JSON line per
log interval plus a summary line.  The fp64 oracle re-check of a final V lives
in tests/test_gpu_parity.py (the oracle is test infrastructure; this tool does
not import it).

  python tools/descent.py --config c2_n10_2d10 --opt adam --lr 3e-3 --steps 20000
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import seeded_inputs as si  # noqa: E402


def planted_target(sos, ix, cfg, seed, dev):
    """p = coef(W W^T) (+ eps (sum x_i^2)^d for config 3), computed by the CUDA path."""
    import torch
    W = torch.from_numpy(si.planted_w(ix.N, cfg.r_star, seed=seed)).to(dev)
    plan_w = sos.SosPlan(ix, cfg.r_star)
    p = plan_w.forward(W)
    torch.cuda.synchronize()
    plan_w.close()
    if cfg.eps:
        sphere = si.sphere_power_coefficients(ix.beta().cpu().numpy(), cfg.d)
        p = (p.double() + cfg.eps * torch.from_numpy(sphere).to(dev)).float()
    return p


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2_n10_2d10", choices=sorted(si.CONFIGS))
    ap.add_argument("--opt", default="adam", choices=["adam", "gd"])
    ap.add_argument("--lr", type=float, default=1e-3)
    ap.add_argument("--steps", type=int, default=20000)
    ap.add_argument("--target", type=float, default=1e-8)
    ap.add_argument("--log-every", type=int, default=250)
    ap.add_argument("--decay", type=float, default=1.0,
                    help="multiply lr by this factor whenever eps_rel rises between log points")
    ap.add_argument("--min-lr", type=float, default=0.0)
    ap.add_argument("--time-limit", type=float, default=1e9, help="seconds")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--save-v", default="")
    args = ap.parse_args()

    import torch
    import paper_2410_19844_b200 as sos

    dev = torch.device("cuda", 0)
    cfg = si.CONFIGS[args.config]
    ix = sos.SosIndex(cfg.n, cfg.d)
    p = planted_target(sos, ix, cfg, args.seed, dev)
    pn = float(torch.dot(p.double(), p.double()).item())
    V0 = si.v0(ix.N, cfg.r, seed=args.seed)
    V = torch.from_numpy(V0).to(dev)
    plan = sos.SosPlan(ix, cfg.r)
    plan.opt_init(args.opt, args.lr)
    plan.set_stop(args.target)  # device-side: V freezes at the first iterate meeting the target
    lr = args.lr
    losses = torch.empty(args.log_every, dtype=torch.float64, device=dev)
    t0 = time.perf_counter()
    prev = math.inf
    hist = []
    step = 0
    reached = None
    while step < args.steps:
        k = min(args.log_every, args.steps - step)
        for u in range(k):
            plan.step(V, p, losses[u:u + 1])
        step += k
        ls = losses[:k].cpu().numpy() / pn   # eps_rel before each of these k updates
        cur = float(ls[-1])
        hit = np.nonzero(ls <= args.target)[0]
        el = time.perf_counter() - t0
        rec = {"step": step, "eps_rel": cur, "min_eps_rel": float(ls.min()), "lr": lr, "s": round(el, 2)}
        hist.append(rec)
        print(json.dumps(rec), flush=True)
        if hit.size:
            reached = step - k + int(hit[0])  # steps taken before the iterate that met the target
            break
        if not math.isfinite(cur) or el > args.time_limit:
            break
        if cur > prev and args.decay < 1.0:
            lr = max(args.min_lr, lr * args.decay)
            plan.set_lr(lr)
        prev = cur
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    # with the device-side stopping rule the final V is the iterate that met
    # the target: re-evaluate its loss (one extra evaluation)
    loss_final, _, _ = plan.loss_grad(V, p, want_grad=False)
    final = float(loss_final.item()) / pn
    out = {"config": cfg.name, "N": ix.N, "M": ix.M, "r": cfg.r, "r_star": cfg.r_star, "opt": args.opt,
           "lr0": args.lr, "lr_final": lr, "decay": args.decay, "steps_run": step,
           "reached_target_at_step": reached, "target": args.target, "eps_rel_final_gpu": final,
           "seconds": round(el, 2), "steps_per_s": step / el}
    if args.save_v:
        np.save(args.save_v, V.cpu().numpy())
    print(json.dumps({"summary": out}), flush=True)


if __name__ == "__main__":
    main()
