#!/usr/bin/env python3
"""Diagnostic: device discriminator gradient (msk_disc_trainer_gradient) vs the f64
oracle per parameter block, for a few shapes.

  python tools/disc_train_check.py [math]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_2603_29332_b200 as pk
    from oracle.disc_train import disc_loss_grad
    from oracle.oracle import mlp_init

    math = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    names = ["W0", "b0", "W1", "b1", "W2", "b2", "w4", "b4"]
    for din, H, B in [(9, 16, 37), (20, 32, 77), (102, 256, 1000), (102, 256, 300)]:
        theta = mlp_init(din, H, 7)
        rng = np.random.default_rng(din + B)
        delta = rng.normal(0, 0.3, (B, din)).astype(np.float32)
        loss, logistic, pen, gref = disc_loss_grad(theta, din, H, delta.astype(np.float64), 10.0)
        tr = pk.DiscTrainer(din, H, theta, lr=1e-3, grad_penalty=10.0, max_rows=B, math=math)
        g, lv = tr.gradient(torch.as_tensor(delta, device="cuda"))
        g, lv = g.cpu().numpy().astype(np.float64), lv.cpu().numpy()
        o, out = 0, []
        for r, c in [(H, din), (H, H), (H, H), (1, H)]:
            for a, b in [(o, o + r * c), (o + r * c, o + r * c + r)]:
                out.append(np.linalg.norm(g[a:b] - gref[a:b]) / max(np.linalg.norm(gref[a:b]), 1e-30))
            o += r * c + r
        print(f"din={din} H={H} B={B} math={math}: loss {lv} ref {[loss, logistic, pen]}")
        print("   " + "  ".join(f"{n} {e:.2e}" for n, e in zip(names, out)))
        tr.close()


if __name__ == "__main__":
    main()
