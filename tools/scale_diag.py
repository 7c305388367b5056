#!/usr/bin/env python3
"""Replays one SCALE_CASES batch (tests/test_gpu.py) and prints, per step, the
worst sampled env's q / q̇ error with its flags, contact forces and power.

    python tools/scale_diag.py c5_wb700_slow_8192 [steps]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch

    import paper_2603_29332_b200 as pk
    from conftest import ensure_assets, model_paths
    from parity_util import f32_state, q_ratio, to_np
    from test_gpu import SCALE_CASES, _gpu_rows
    from oracle.oracle import OracleBatch, excitations
    from oracle.ref import env_config

    ensure_assets()
    case = sys.argv[1]
    model, E, cfg_kw, mode, disc, ev, steps, h = SCALE_CASES[case]
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else steps
    mp, cp = model_paths(model)
    g = pk.EnvBatch(mp, cp, E, cfg=pk.EnvConfig(**cfg_kw), reward=pk.RewardConfig(mode=mode))
    g.set_eval_mode(ev)
    rng = np.random.default_rng(11)
    sample = [0, 1, E - 1] + sorted(rng.choice(np.arange(2, E - 1), 13, replace=False).tolist())
    orc = {}
    for e in sample:
        o = OracleBatch(mp, cp, 1, cfg=env_config(**cfg_kw), reward_mode=mode, global_env_offset=e)
        o.set_eval_mode(ev)
        orc[e] = o
    g.reset()
    for o in orc.values():
        o.reset()
    a = torch.empty(E, g.nm, device=g.device)
    for s in range(steps):
        pre = _gpu_rows(g, sample)
        for k, (e, o) in enumerate(orc.items()):
            o.set_state(f32_state({kk: v[k:k + 1] for kk, v in pre.items()}) | {"ints": pre["ints"][k:k + 1]})
        g.fill_excitations(0x5EED, s, a)
        out = g.step(a, want_power=True, want_contact=True)
        post = _gpu_rows(g, sample)
        fl = to_np(out["flags"])
        cf = to_np(out["contact_force"])
        for k, (e, o) in enumerate(orc.items()):
            oo = o.step(excitations(0x5EED, s, 1, g.nm, global_env_offset=e))
            so = o.get_state()
            rq, rd = q_ratio(post["q"][k], so["q"][0]), q_ratio(post["dq"][k], so["dq"][0])
            dd_ = np.abs(post["dq"][k] - so["dq"][0])
            i_ = int(np.argmax(dd_ / np.maximum(1e-3 * np.abs(so["dq"][0]), 5e-5)))
            print(f"  step {s} env {e}: max|q̇| {np.abs(so['dq'][0]).max():.3g} (dof {int(np.argmax(np.abs(so['dq'][0])))}),"
                  f" worst dof {i_}: |d| {dd_[i_]:.3g} ref {so['dq'][0][i_]:.4g}; max|d| {dd_.max():.3g}")
            if rq > 1 or rd > 1:
                grf_o = np.asarray(oo["grf"]).reshape(-1)
                dd = np.abs(cf[e].reshape(-1) - grf_o)
                print(f"step {s} env {e} flags {fl[e]} t_index {pre['ints'][k]}: q ratio {rq:.3g} dq ratio {rd:.3g}; "
                      f"grf max|d| {dd.max():.3g} at {np.argmax(dd)} (gpu {cf[e].reshape(-1)[np.argmax(dd)]:.4g}, ref "
                      f"{grf_o[np.argmax(dd)]:.4g}); gpu grf nonzero {np.nonzero(np.abs(cf[e].reshape(-1)) > 0)[0].tolist()}")
        done = (fl & 1) > 0
        if h and (s + 1) % h == 0:
            bins, failed, counts = g.drain_outcomes(h)
            g.merge_outcomes(bins, failed, counts)
            ema = to_np(g.get_sampler())[0]
            for o in orc.values():
                o.drain_outcomes(h)
                o.set_sampler(ema[None, :])
        if done.any():
            g.reset(mask=out["flags"], mask_bits=pk.FLAG_DONE)
            for e, o in orc.items():
                if done[e]:
                    o.reset()
    g.close()


if __name__ == "__main__":
    main()
