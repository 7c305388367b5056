#!/usr/bin/env python3
"""Times the on-device discriminator training step (msk_disc_train_step) on a
c4-sized batch: h*E = 8 * 16384 Delta rows of the wb700 model (dΔ = 102), W = 256.

  python tools/disc_train_bench.py [rows] [math] [iters]
Prints one JSON line: ms per step, algorithmic GFLOP per step and TFLOP/s."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def flops(B, din, H):
    """GEMM flops of one step (2 m n k each): forward 3 + head, d-chain 3, tangent 3 + head,
    reverse weight grads over 2R rows (3 + head), reverse adjoint products over 2R rows (2)."""
    R = B + 1
    fwd = 2 * R * (din * H + 2 * H * H + H)
    dchain = 2 * R * (2 * H * H + H * din)
    tangent = 2 * R * (din * H + 2 * H * H + H)
    wgrad = 2 * (2 * R) * (din * H + 2 * H * H + H)
    adj = 2 * (2 * R) * (2 * H * H)
    return fwd + dchain + tangent + wgrad + adj


def main():
    import torch

    import paper_2603_29332_b200 as pk

    B = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
    math = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    iters = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    din, H = 102, 256
    tr = pk.DiscTrainer(din, H, pk.mlp_init(din, H, 7), lr=3e-5, grad_penalty=10.0, max_rows=B, math=math)
    delta = torch.randn(B, din, device="cuda") * 0.2
    for _ in range(3):
        tr.step(delta)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        tr.step(delta)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    f = flops(B, din, H)
    print(json.dumps({"rows": B, "din": din, "hidden": H, "math": ["fp32-class split-bf16", "bf16"][math], "ms_per_step": ms,
                      "gflop_per_step": f / 1e9, "tflops": f / (ms * 1e-3) / 1e12,
                      "loss": tr.loss.cpu().tolist()}))
    tr.close()


if __name__ == "__main__":
    main()
