#!/usr/bin/env python3
"""Per-phase cycle breakdown of the step kernel (needs a -DMSK_PHASE_TIMERS build in $MSK_B200_LIB)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_29332_b200 as pk  # noqa: E402
from tools.gen_assets import generate  # noqa: E402

NAMES = ["muscles", "torques", "sweep(FK+vel+ABA init)", "ABA leaf->root", "root solve + ABA root->leaf",
         "integrate+publish"]


def main():
    d = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "assets", "generated")
    if not os.path.exists(os.path.join(d, "wb700_fixed.json")):
        generate(d)
    model = sys.argv[1] if len(sys.argv) > 1 else "wb700_fixed"
    clip = {"wb700_fixed": "wb700_fixed_dance", "wb700": "wb700_dance"}[model]
    E = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
    env = pk.EnvBatch(os.path.join(d, model + ".json"), os.path.join(d, clip + ".csv"), E,
                      cfg=pk.EnvConfig(episode_horizon=1000, rsi=False))
    env.set_eval_mode(True)
    env.reset()
    L = pk.lib()
    L.msk_gpu_phase_cycles.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
    buf = (C.c_ulonglong * 8)()
    a = env.fill_excitations(1, 0)
    for s in range(3):
        env.step(a)
    torch.cuda.synchronize()
    L.msk_gpu_phase_cycles(buf, 1)
    steps = 5
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for s in range(steps):
        env.step(a)
    ev1.record()
    torch.cuda.synchronize()
    L.msk_gpu_phase_cycles(buf, 1)
    tot = sum(buf[:6])
    per = E * steps * 10
    print(f"{model} E={E}: {ev0.elapsed_time(ev1) / steps:.3f} ms/step; cycles per warp-substep total {tot / per:.0f}")
    for i, n in enumerate(NAMES):
        print(f"  {n:32s} {buf[i] / per:8.0f} cycles  {buf[i] / tot * 100:5.1f}%")


if __name__ == "__main__":
    main()
