#!/usr/bin/env python3
"""Generates the golden fixtures from the REFERENCE itself.

Runs the reference's own msk::Env (oracle/_ref/libmsk_ref.so, compiled
unchanged from /root/reference/proj/src by oracle/Makefile) on seeded inputs
and stores what it produced, so the parity tests on machines without
/root/reference (the GPU box) still check against reference output.

    python tests/golden/make_golden.py      # writes tests/golden/*.npz

Each fixture holds, for E envs of one model/clip: the start frames of two
rounds of RSI resets, the excitations, and after every control step the
flags, Δ, observation, reward_aux and the full state (q, dq, act, l_m, v_m,
f_m, t, t_index/start/steps/done), plus raw mt19937_64 draws and the sampler.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from conftest import ensure_assets, model_paths  # noqa: E402
from oracle.ref import RefBatch, env_config, excitations  # noqa: E402

from golden_cases import CASES  # noqa: E402


def make(name):
    n, steps, cfg_kw, mode = CASES[name]
    mp, cp = model_paths(name)
    b = RefBatch(mp, cp, n, base_seed=0x5EED, cfg=env_config(**cfg_kw), reward_mode=mode)
    # a non-trivial sampler so RSI exercises the failure-proportional branch
    ema = np.linspace(0.0, 0.3, b.bins)[None, :] * (1 + np.arange(n)[:, None] * 0.1)
    b.set_sampler(ema)
    obs0, frames0 = b.reset()
    rec = dict(frames0=frames0, obs0=obs0, ema0=ema)
    keys = ("flags", "delta", "obs", "reward_aux", "power")
    hist = {k: [] for k in keys}
    shist = {k: [] for k in ("q", "dq", "act", "l_m", "v_m", "f_m", "t", "ints")}
    acts, reset_frames = [], []
    for s in range(steps):
        a = excitations(0xA11CE, s, n, b.nm)
        acts.append(a)
        r = b.step(a)
        for k in keys:
            hist[k].append(r[k])
        st = b.get_state()
        for k in shist:
            shist[k].append(st[k])
        done = (r["flags"] & 1).astype(np.uint8)
        fr = np.full(n, -1, dtype=np.int32)
        if done.any():
            b.record_own_outcomes()
            _, f = b.reset(mask=done)
            fr = np.where(done > 0, f, -1)
        reset_frames.append(fr)
    rec.update({k: np.stack(v) for k, v in hist.items()})
    rec.update({"state_" + k: np.stack(v) for k, v in shist.items()})
    rec["actions"] = np.stack(acts)
    rec["reset_frames"] = np.stack(reset_frames)
    rec["ema_end"] = b.get_sampler()
    rec["rng_draws"] = b.rng_raw(0, 400)  # crosses a 312-word twist
    rec["meta"] = np.array([n, steps, mode], dtype=np.int64)
    return rec


def mlp_theta_from_reference_rng(n_in, hidden, seed, n_out=1, final_init_scale=1.0):
    """Mlp::Mlp(shape, seed) weights (nn.cpp:16-38) from the reference's OWN
    msk::Rng(seed) uniform stream: uniform(lo, hi) = lo + (hi - lo) * uniform()
    (rng.hpp:26-30), column-major per layer, biases zero."""
    from oracle.ref import rng_uniform

    dims = [(hidden, n_in), (hidden, hidden), (hidden, hidden), (n_out, hidden)]
    n_w = sum(r * c for r, c in dims)
    u = rng_uniform(seed, 0.0, 1.0, n_w)  # lo + (1 - 0) * u == u exactly
    theta, k = [], 0
    for layer, (r, c) in enumerate(dims):
        s = (1.0 / np.sqrt(float(c))) * (final_init_scale if layer == 3 else 1.0)
        w = -s + (s - -s) * u[k:k + r * c]
        k += r * c
        theta += [w, np.zeros(r)]
    return np.concatenate(theta)


def make_mlp():
    small = mlp_theta_from_reference_rng(9, 16, 7)
    big = mlp_theta_from_reference_rng(102, 256, 7)
    return dict(small=small, big_head=big[:512], big_tail=big[-512:], big_sum=np.array([np.sum(big)]),
                big_len=np.array([big.size]))


RNG_CASE = dict(model="arm2_m6", n=3, rounds=5, cfg=dict(episode_horizon=30, rsi=True))


def make_rng():
    """The reference's own Rng::serialize() text (rng.hpp:56-61) of every env at
    construction and after each of `rounds` RSI resets of all envs, plus the
    start frames of every round (Env::rng(), env.hpp:120)."""
    c = RNG_CASE
    mp, cp = model_paths(c["model"])
    b = RefBatch(mp, cp, c["n"], base_seed=0x5EED, cfg=env_config(**c["cfg"]))
    ema = np.linspace(0.0, 0.3, b.bins)
    b.set_sampler(np.tile(ema, (c["n"], 1)))
    states = [[b.rng_serialize(e) for e in range(c["n"])]]
    frames = []
    for _ in range(c["rounds"]):
        _, f = b.reset()
        frames.append([int(x) for x in f])
        states.append([b.rng_serialize(e) for e in range(c["n"])])
    return dict(case=c, ema=ema.tolist(), serialize=states, frames=frames)


def make_nn():
    """The reference's own nn.cpp (Mlp::forward / backward / gradient_penalty_backward)
    on a fixed small case (tests/test_disc_train.py::_nn_case)."""
    from oracle.oracle import mlp_init
    from oracle.ref import ref_mlp_backward, ref_mlp_forward, ref_mlp_gp_backward

    din, H, B = 9, 16, 7
    rng = np.random.default_rng(11)
    theta = mlp_init(din, H, 3)
    theta = theta + rng.normal(0, 0.05, theta.shape)
    X = rng.normal(0, 0.8, (B, din))
    up = rng.normal(0, 1.0, (B, 1))
    gb, ig = ref_mlp_backward(theta, din, H, 1, X, up)
    gp, pen = ref_mlp_gp_backward(theta, din, H, X)
    return dict(shape=np.array([din, H]), theta=theta, X=X, up=up, y=ref_mlp_forward(theta, din, H, 1, X),
                grad_backward=gb, input_grad=ig, grad_penalty=gp, penalty=pen)


def main():
    ensure_assets()
    import json

    path = os.path.join(HERE, "nn_reference.npz")
    np.savez_compressed(path, **make_nn())
    print(path, os.path.getsize(path))

    path = os.path.join(HERE, "rng_serialize.json")
    with open(path, "w") as f:
        json.dump(make_rng(), f)
    print(path, os.path.getsize(path))
    path = os.path.join(HERE, "mlp_seed7.npz")
    np.savez_compressed(path, **make_mlp())
    print(path, os.path.getsize(path))
    for name in CASES:
        rec = make(name)
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **rec)
        print(path, os.path.getsize(path))


if __name__ == "__main__":
    main()
