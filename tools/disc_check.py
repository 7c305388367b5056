#!/usr/bin/env python3
"""GPU check of the tensor-core discriminator against the f64 oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_29332_b200 as pk  # noqa: E402
from oracle.oracle import disc_reward, mlp_init  # noqa: E402
from tools.gen_assets import generate  # noqa: E402


def main():
    d = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "assets", "generated")
    if not os.path.exists(os.path.join(d, "wb700.json")):
        generate(d)
    env = pk.EnvBatch(os.path.join(d, "wb700.json"), os.path.join(d, "wb700_dance.csv"), 256)
    dd = env.delta_dim
    rng = np.random.default_rng(0)
    for H in (16, 64, 256):
        for fis in (1.0, 0.0):
            th = mlp_init(dd, H, 7, final_init_scale=fis)
            env.set_discriminator(th, H)
            for scale in (0.05, 0.3, 1.0, 3.0):
                x = rng.normal(0, scale, (300, dd)).astype(np.float32)
                r = env.discriminator_reward(torch.as_tensor(x, device="cuda"))
                torch.cuda.synchronize()
                ref = disc_reward(th, dd, H, x.astype(np.float64))
                e = np.abs(r.cpu().numpy() - ref)
                print(f"H={H:3d} fis={fis} scale={scale:4.2f}: max|dr|={e.max():.3e} rel={np.max(e / ref):.3e} "
                      f"r=[{ref.min():.4f},{ref.max():.4f}]")
    env.close()


if __name__ == "__main__":
    main()
