"""Debug: smoke's wb700 control step on the device only; saves the state to argv[1]."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import ensure_assets, model_paths
from parity_util import gpu_state, make_pair, sync_from_oracle
from oracle.oracle import excitations
ensure_assets()
mp, cp = model_paths("wb700")
n = 4
g, o = make_pair(mp, cp, n, cfg_kw=dict(episode_horizon=1000, rsi=False))
g.reset_to_frame(np.arange(n) * 11); o.reset_to_frame(np.arange(n) * 11)
sync_from_oracle(g, o)
a = excitations(0x5EED, 0, n, g.nm).astype(np.float32)
out = []
for k in range(1, 11):
    st = g.get_state()
    g.substeps(torch.as_tensor(a, device=g.device), k) if k < 10 else g.step(torch.as_tensor(a, device=g.device))
    torch.cuda.synchronize()
    out.append(gpu_state(g)["dq"])
    g.set_state(st)
np.save(sys.argv[1], np.array(out))
