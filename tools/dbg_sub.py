"""Debug: one substep from identical state, per-DOF qdd error vs the oracle (device ABA + torques)."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import ensure_assets, model_paths
from parity_util import gpu_state, make_pair, sync_from_oracle
from oracle.oracle import excitations
ensure_assets()
name = sys.argv[1] if len(sys.argv) > 1 else "wb700"
mp, cp = model_paths(name)
n = 4
g, o = make_pair(mp, cp, n, cfg_kw=dict(episode_horizon=1000, rsi=False))
g.reset_to_frame(np.arange(n) * 11); o.reset_to_frame(np.arange(n) * 11)
s0 = sync_from_oracle(g, o)
a = excitations(0x5EED, 0, n, g.nm).astype(np.float32)
g.substeps(torch.as_tensor(a, device=g.device), 1)
torch.cuda.synchronize()
sg = gpu_state(g)
# oracle single substep per env
m = o.model
err = np.zeros((n, sg["dq"].shape[1]))
for e in range(n):
    st = {k: np.asarray(s0[k][e]) for k in ("q", "dq", "act", "l_m", "v_m", "f_m")}
    u = np.clip(a[e].astype(np.float64), 0, 1)
    ns, _, bad = m.substep(st["q"], st["dq"], st["act"], st["l_m"], st["v_m"], st["f_m"], u)
    err[e] = (sg["dq"][e] - ns["dq"]) / 0.002
np.set_printoptions(precision=3, linewidth=200)
top = np.argsort(-np.abs(err).max(0))[:8]
print("top DOFs by |qdd err|:", top, np.abs(err).max(0)[top])
print("max |qdd err|", np.abs(err).max())
g.close()
