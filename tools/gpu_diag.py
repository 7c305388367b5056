#!/usr/bin/env python3
"""GPU-vs-oracle error survey (prints per-model single-step and short-horizon errors).

    python tools/gpu_diag.py [steps]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from conftest import ensure_assets, model_paths  # noqa: E402
from parity_util import f32_state, force_err, gpu_state, make_pair, rel_err, step_both, sync_from_oracle  # noqa: E402
from oracle.oracle import excitations  # noqa: E402


def main():
    import torch

    ensure_assets()
    horizon = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    for name, n in (("pendulum1_m2", 4), ("arm2_m6", 8), ("walker5_m16", 8), ("wb700_fixed", 4), ("wb700", 4),
                    ("wb700_backflip", 4)):
        mp, cp = model_paths(name)
        t0 = time.time()
        g, o = make_pair(mp, cp, n, cfg_kw=dict(episode_horizon=1000, rsi=False))
        g.set_eval_mode(True)
        o.set_eval_mode(True)
        frames = np.arange(n) * 37 % (o.frames - 2)
        g.reset_to_frame(frames)
        o.reset_to_frame(frames)
        torch.cuda.synchronize()
        sg, so = gpu_state(g), o.get_state()
        print(f"== {name}: reset q err {np.abs(sg['q'] - so['q']).max():.2e} l_m rel err "
              f"{rel_err(sg['l_m'], so['l_m'], 1e-3):.2e} f_m/fmax err "
              f"{force_err(sg['f_m'], so['f_m'], o.model.d['m_fmax']):.2e}")
        fmax = o.model.d["m_fmax"]
        worst = {}
        for s in range(horizon):
            sync_from_oracle(g, o) if s == 0 or "--resync" in sys.argv else None
            a = excitations(0x5EED, s, n, o.nm).astype(np.float32)
            og, oo = step_both(g, o, a)
            sg, so = gpu_state(g), o.get_state()
            errs = dict(
                q=np.abs(sg["q"] - so["q"]).max() / max(1.0, np.abs(so["q"]).max()),
                dq=np.abs(sg["dq"] - so["dq"]).max() / max(1.0, np.abs(so["dq"]).max()),
                act=np.abs(sg["act"] - so["act"]).max(),
                f=force_err(sg["f_m"], so["f_m"], fmax),
                obs=np.abs(og["obs"] - oo["obs"]).max() / max(1.0, np.abs(oo["obs"]).max()),
                delta=np.abs(og["delta"] - oo["delta"]).max(),
                flags=int((og["flags"] != oo["flags"]).sum()),
                power=np.abs(og["muscle_power"] - oo["power"]).max() / max(1.0, np.abs(oo["power"]).max()),
                grf=np.abs(og["contact_force"] - oo["grf"]).max() / max(1.0, np.abs(oo["grf"]).max()),
            )
            if s in (0, horizon - 1):
                print(f"  step {s:3d}: " + " ".join(f"{k}={v:.2e}" if isinstance(v, float) else f"{k}={v}"
                                                      for k, v in errs.items()))
            for k, v in errs.items():
                worst[k] = max(worst.get(k, 0), v)
        print("  worst: " + " ".join(f"{k}={v:.2e}" for k, v in worst.items()), f"({time.time() - t0:.1f}s)")
        g.close()


if __name__ == "__main__":
    main()
