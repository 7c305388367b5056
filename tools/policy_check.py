#!/usr/bin/env python3
"""Paper-scale policy sampling on one GPU: timing (CUDA graph replay) and error vs the f64 oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_29332_b200 as pk  # noqa: E402
from oracle.policy import sample_action  # noqa: E402


def main():
    D, NM = 3106, 700
    H = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    E = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
    n_ode = 20
    pi = pk.mlp_init(D, H, 1, n_out=NM, final_init_scale=0.01)
    psi = pk.mlp_init(5 + D + NM, H, 2, n_out=NM, final_init_scale=0.01)
    ls = np.full(NM, -1.0)
    p = pk.Policy(D, NM, H, pi, ls, psi, n_ode=n_ode, max_envs=E, head_offset=0.5)
    rng = np.random.default_rng(0)
    obs = torch.as_tensor(rng.normal(0, 1, (E, D)).astype(np.float32), device="cuda")
    act = torch.empty(E, NM, device="cuda")
    for _ in range(3):
        p.sample(obs, explore=True, seed=1, step=0, actions=act, graph=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        p.sample(obs, explore=True, seed=1, step=0, actions=act, graph=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    Kp = lambda k: (k + 63) // 64 * 64  # noqa: E731
    flops = 2.0 * E * (Kp(D) * H + 2 * H * H + H * NM) + 2.0 * E * Kp(D) * H \
        + n_ode * 2.0 * E * (Kp(NM) * H + 2 * H * H + H * NM)
    print(f"H={H} E={E} n_ode={n_ode}: {ms:.3f} ms per sample, {flops / ms / 1e9:.1f} TFLOP/s "
          f"({flops / E / 1e6:.1f} MFLOP per env)")
    # accuracy on a slice
    n = 64
    a = p.sample(obs[:n]).cpu().numpy()
    ref, _, _ = sample_action(pi, ls, psi, obs[:n].cpu().numpy(), H, n_ode=n_ode, head_offset=0.5)
    print(f"max |a - a_f64| = {np.abs(a - ref).max():.3e}  (|a| max {np.abs(ref).max():.3f})")
    p.close()


if __name__ == "__main__":
    main()
