"""Debug: smoke's wb700 step, per-quantity error ratios (power on / off, 1 substep / control step)."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import ensure_assets, model_paths
from parity_util import f_ratio, gpu_state, make_pair, q_ratio, sync_from_oracle
from oracle.oracle import excitations
ensure_assets()
name = sys.argv[1] if len(sys.argv) > 1 else "wb700"
mp, cp = model_paths(name)
n = 4
for want_power in (False, True):
    g, o = make_pair(mp, cp, n, cfg_kw=dict(episode_horizon=1000, rsi=False))
    g.reset_to_frame(np.arange(n) * 11); o.reset_to_frame(np.arange(n) * 11)
    sync_from_oracle(g, o)
    a = excitations(0x5EED, 0, n, g.nm).astype(np.float32)
    g.step(torch.as_tensor(a, device=g.device), want_power=want_power, want_contact=True)
    torch.cuda.synchronize()
    o.step(a.astype(np.float64))
    sg, so = gpu_state(g), o.get_state()
    for k in ("q", "dq"):
        d = np.abs(sg[k] - so[k]) / np.maximum(1e-5 * np.abs(so[k]), 1e-6)
        i = np.unravel_index(np.argmax(d), d.shape)
        print(f"power={want_power} {k}: ratio {d.max():.3f} at {i} gpu {sg[k][i]:.9g} ref {so[k][i]:.9g}")
    print("  force ratio", f_ratio(sg["f_m"], so["f_m"], o.model.d["m_fmax"]), "act", np.abs(sg["act"] - so["act"]).max())
    g.close()
