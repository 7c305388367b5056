#!/usr/bin/env python3
"""Where do the per-element q / q̇ errors of one control step come from?

Prints the worst DOFs (|Δ|, the reference value, the step's change, the
link's mass / inertia / depth) for a model's single-step parity trial.

    python tools/parity_diag.py wb700_fixed [n_envs]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from conftest import ensure_assets, model_paths  # noqa: E402
from parity_util import f32_state, gpu_state, make_pair, step_both  # noqa: E402
from oracle.oracle import excitations  # noqa: E402


def main():
    import torch

    ensure_assets()
    name = sys.argv[1] if len(sys.argv) > 1 else "wb700_fixed"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    mp, cp = model_paths(name)
    js = json.load(open(mp))
    fc = 1 if js["root"] == "floating" else 0
    nrd = 3 if fc else 0
    parent = [-1] * len(js["links"])
    for j, jt in enumerate(js["joints"]):
        parent[fc + j] = jt["parent"]
    depth = []
    for l in range(len(parent)):
        depth.append(0 if parent[l] < 0 else depth[parent[l]] + 1)
    g, o = make_pair(mp, cp, n, cfg_kw=dict(episode_horizon=1000, rsi=False))
    g.set_eval_mode(True)
    o.set_eval_mode(True)
    frames = (np.arange(n) * 97 + 13) % (o.frames - 2)
    for trial in range(3):
        g.reset_to_frame(frames + trial)
        o.reset_to_frame(frames + trial)
        torch.cuda.synchronize()
        s = o.get_state()
        rng = np.random.default_rng(trial)
        s["dq"] = s["dq"] + rng.normal(0, 0.3, s["dq"].shape)
        s["act"] = rng.uniform(0, 1, s["act"].shape)
        s = f32_state(s)
        o.set_state(s)
        g.set_state(s)
        dq0 = s["dq"].copy()
        a = excitations(1000 + trial, 0, n, g.nm).astype(np.float32)
        step_both(g, o, a)
        sg, so = gpu_state(g), o.get_state()
        for k in ("q", "dq"):
            d = np.abs(sg[k] - so[k])
            ratio = d / np.maximum(1e-5 * np.abs(so[k]), 1e-6)
            order = np.argsort(ratio.ravel())[::-1][:8]
            print(f"{name} trial {trial} {k}: worst ratio {ratio.max():.2f}  (max |d| {d.max():.3g}, "
                  f"max rel-to-row-max {(d.max(1) / np.abs(so[k]).max(1)).max():.3g})")
            for idx in order:
                e, i = divmod(int(idx), so[k].shape[1])
                link = (i - nrd + fc) if i >= nrd else 0
                lk = js["links"][link]
                chg = so["dq"][e, i] - dq0[e, i]
                print(f"   env {e} dof {i:3d} ({lk['name']:>14s}, m {lk['mass']:.3g}, I {lk['inertia']:.2g}, depth "
                      f"{depth[link]:2d}): |d| {d[e, i]:.3g}  ref {so[k][e, i]: .4g}  ratio {ratio[e, i]:.2f}  "
                      f"step dq change {chg: .3g}")
    g.close()


if __name__ == "__main__":
    main()
