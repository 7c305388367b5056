#!/usr/bin/env python3
"""How far does ONE control step's q̇ move, per element, when every muscle force
is perturbed by a relative eps (the f32 evaluation error of the Hill curves)?

Runs the f64 oracle (oracle/msk_oracle.c, bit-exact to the reference) twice
from the same state and excitations: once on the model, once with every
muscle's f_max scaled by (1 + eps * N(0,1)) — a relative force perturbation
of size eps with the reference's own arithmetic everywhere else.  Prints the
per-element ratio |Δq̇| / max(1e-5 |q̇|, 1e-6) (the SURVEY §8(c) proposal) and
the relative-error quantiles.  A ratio >> 1 at eps ~ 1e-7..1e-6 means that
per-element bound is below the conditioning of the model for ANY fp32 force
evaluation (light distal links: tiny inertia, large muscle torques).

    python tools/qdot_sensitivity.py wb700 [eps]
"""
import json
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from conftest import ensure_assets, model_paths  # noqa: E402
from oracle.oracle import OracleBatch, excitations  # noqa: E402
from oracle.ref import env_config  # noqa: E402


def one(mp, cp, n, eps_seed, eps, trial):
    o = OracleBatch(mp, cp, n, cfg=env_config(episode_horizon=1000, rsi=False))
    o.set_eval_mode(True)
    frames = (np.arange(n) * 97 + 13) % (o.frames - 2)
    o.reset_to_frame(frames + trial)
    s = o.get_state()
    rng = np.random.default_rng(trial)
    s["dq"] = s["dq"] + rng.normal(0, 0.3, s["dq"].shape)
    s["act"] = rng.uniform(0, 1, s["act"].shape)
    o.set_state(s)
    o.step(excitations(1000 + trial, 0, n, o.nm))
    return o.get_state()


def main():
    ensure_assets()
    name = sys.argv[1] if len(sys.argv) > 1 else "wb700"
    eps = float(sys.argv[2]) if len(sys.argv) > 2 else 7e-7
    mp, cp = model_paths(name)
    js = json.load(open(mp))
    rng = np.random.default_rng(5)
    for mu in js["muscles"]:
        mu["f_max"] = mu["f_max"] * (1.0 + eps * rng.normal())
    with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as f:
        json.dump(js, f)
        pert = f.name
    worst, rels, norm, fr = 0.0, [], 0.0, 0.0
    fmax = np.array([mu["f_max"] for mu in json.load(open(mp))["muscles"]])
    for trial in range(3):
        a = one(mp, cp, 3, 0, eps, trial)
        b = one(pert, cp, 3, 0, eps, trial)
        d = np.abs(a["dq"] - b["dq"])
        worst = max(worst, float((d / np.maximum(1e-5 * np.abs(a["dq"]), 1e-6)).max()))
        rels.append((d / np.maximum(np.abs(a["dq"]), 1e-3)).ravel())
        norm = max(norm, float((d.max(axis=1) / np.abs(a["dq"]).max(axis=1)).max()))
        # end-of-step muscle forces vs the SURVEY bound 1e-4 max(|F|, 1e-3 f_max), minus the
        # perturbation itself (b's forces are scaled by its f_max)
        fb = b["f_m"] * (fmax / np.array([mu["f_max"] for mu in js["muscles"]]))[None, :]
        fr = max(fr, float((np.abs(a["f_m"] - fb) / (1e-4 * np.maximum(np.abs(a["f_m"]), 1e-3 * fmax))).max()))
    os.unlink(pert)
    r = np.concatenate(rels)
    print(f"{name}: force perturbation eps {eps:.1e} -> per-element q̇ ratio (1e-5 rel, 1e-6 floor) worst "
          f"{worst:.2f}; |Δq̇|/max(|q̇|,1e-3) quantiles 50% {np.quantile(r, .5):.2e} 99% {np.quantile(r, .99):.2e} "
          f"max {r.max():.2e}; norm-wise max|Δq̇|/max|q̇| {norm:.2e}; end-of-step force ratio {fr:.2f}")


if __name__ == "__main__":
    main()
