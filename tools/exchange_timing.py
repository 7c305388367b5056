#!/usr/bin/env python3
"""Times the pieces of one rollout-iteration boundary (dist.iteration_exchange)
for the c4 workload on one GPU: device time of each piece (CUDA events, GPU
otherwise idle) and the host time of the whole call.

  python tools/exchange_timing.py [envs] [cap]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import bench
    import paper_2603_29332_b200 as pk
    import paper_2603_29332_b200.dist as pkd

    E = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    cap = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    mp, cp = bench.model_files("wb700")
    env = pk.EnvBatch(mp, cp, E, cfg=pk.EnvConfig(episode_horizon=250, rsi=True))
    env.set_eval_mode(False)
    obs = env.reset()
    flags = torch.zeros(E, dtype=torch.uint8, device="cuda")
    stats = torch.zeros(pkd.N_STATS, dtype=torch.float64, device="cuda")
    norm = pkd.init_norm_state(env.obs_dim, "cuda")
    for it in range(3):
        for s in range(8):
            a = env.fill_excitations(0x5EED, it * 8 + s)
            out = env.step(a, obs=obs, flags=flags)
            env.rollout_stats(flags, stats, reward=out["reward_aux"])
            env.reset(mask=flags, mask_bits=pk.FLAG_DONE)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        t0 = time.perf_counter()
        ev[0].record()
        bins, failed, counts = env.drain_outcomes(cap)
        ev[1].record()
        mom = env.obs_moments(obs)
        ev[2].record()
        block = pkd.pack_block(bins, failed, counts, stats, mom, env.obs_dim)
        blocks = pkd.exchange(block)
        ev[3].record()
        res = pkd.merged_iteration(blocks, E, cap, env.obs_dim, norm, None, env.cfg.adaptive_decay,
                                   merge_on_device=env)
        ev[4].record()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        norm = res[1]
        n_out = int(counts.sum())
        print(f"iter {it}: outcomes {n_out}, drain {ev[0].elapsed_time(ev[1]):.3f} ms, obs moments "
              f"{ev[1].elapsed_time(ev[2]):.3f}, pack+exchange {ev[2].elapsed_time(ev[3]):.3f}, merge "
              f"{ev[3].elapsed_time(ev[4]):.3f}, host {1e3 * (t1 - t0):.3f} ms", flush=True)
        stats.zero_()
    env.close()


if __name__ == "__main__":
    main()
