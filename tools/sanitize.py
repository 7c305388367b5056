#!/usr/bin/env python3
"""Small-E workload that launches every kernel of libmsk_b200.so once or twice
(ragged env counts 5 / 29 — not multiples of the 28-env block or 32-lane
chunks; every model family: fixed / floating, contacts, generic segments; the
rewarded step (tcgen05 discriminator), host-buffer step, reset paths, state
I/O, outcome drain / merge, reductions, policy sampling (tcgen05 GEMM),
rollout buffer + GAE and the discriminator training step).

It was written for compute-sanitizer, which this GPU pool
has closed (runs under it left GPUs needing a reset); it runs plain as a
coverage smoke test, and the out-of-bounds question is answered by the guard-
zone test tests/test_gpu.py::test_outputs_stay_inside_caller_buffers.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch

    import paper_2603_29332_b200 as pk
    from conftest import ensure_assets, model_paths

    ensure_assets()
    for name, n in (("arm2_m6", 5), ("walker5_m16", 29), ("wb700", 5)):
        mp, cp = model_paths(name)
        env = pk.EnvBatch(mp, cp, n, cfg=pk.EnvConfig(episode_horizon=3),
                          reward=pk.RewardConfig(mode=pk.RewardMode.ImitationPower))
        obs = env.reset()
        actions = torch.rand(n, env.nm, device="cuda")
        if name == "wb700":
            env.set_discriminator(pk.mlp_init(env.delta_dim, 64, 7), 64)
        for s in range(4):  # the horizon of 3 ends episodes inside the loop
            out = env.step(actions, reward=torch.zeros(n, device="cuda") if name == "wb700" else None,
                           want_power=True, want_contact=True)
            env.reset(mask=out["flags"], mask_bits=pk.FLAG_DONE)
        env.fill_excitations(0x5EED, 1, actions)
        env.observe()
        env.tracking_error()
        env.force_state_to_reference()
        st = env.get_state()
        env.set_state(st)
        env.reset_to_frame(torch.arange(n, dtype=torch.int32, device="cuda"))
        stats = torch.zeros(7, dtype=torch.float64, device="cuda")
        env.rollout_stats(out["flags"], stats, reward=out["reward_aux"])
        env.obs_moments(obs)
        bins, failed, counts = env.drain_outcomes()
        env.merge_outcomes(bins, failed, counts)
        env.get_sampler()
        env.rng_raw(0, 4)
        ah = torch.rand(n, env.nm).pin_memory()
        env.step_host(ah, torch.empty(n, env.obs_dim).pin_memory(), torch.empty(n, env.delta_dim).pin_memory(),
                      torch.empty(n).pin_memory(), torch.empty(n, dtype=torch.uint8).pin_memory())
        if name == "wb700":
            W = 64
            pol = pk.Policy(env.obs_dim, env.nm, W, pk.mlp_init(env.obs_dim, W, 1, n_out=env.nm),
                            [-1.0] * env.nm, pk.mlp_init(5 + env.obs_dim + env.nm, W, 2, n_out=env.nm), n_ode=2,
                            max_envs=n)
            a0 = torch.empty(n, env.nm, device="cuda")
            lp = torch.empty(n, device="cuda")
            pol.sample(obs, explore=True, seed=1, step=0, actions=actions, a0=a0, logprob=lp)
            ro = pk.Rollout(n, 2, env.obs_dim, env.nm, env.delta_dim)
            for t in range(2):
                out = env.step(actions)
                ro.record(t, obs=obs, a0=a0, actions=actions, logprob=lp, reward=out["reward_aux"],
                          flags=out["flags"], value=torch.zeros(n, device="cuda"), delta=out["delta"])
            ro.gae(torch.zeros(n, device="cuda"))
            tr = pk.DiscTrainer(env.delta_dim, 64, pk.mlp_init(env.delta_dim, 64, 7), max_rows=2 * n)
            tr.step(ro.field(7, env.delta_dim))
            tr.publish(env)
            pol.close()
            ro.close()
            tr.close()
        torch.cuda.synchronize()
        env.close()
        print(f"{name}: ok", flush=True)


if __name__ == "__main__":
    main()
