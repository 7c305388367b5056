"""Oracle (test infrastructure only): f64 restatement of the policy sampler.

sample_action: a0 = mean(s) (+ exp(log_std) * eps when
exploring), then a = a0 + sum_k psi(k dt, s, a_k) dt by explicit Euler over
N_ODE steps.  mean = head_scale * Mlp_pi(norm(s)) + head_offset (Head::Affine,
nn.hpp:10-19); psi = Mlp_psi([phi(t), norm(s), a]) with the time features
phi(t) = [t, sin 2 pi t, cos 2 pi t, sin 4 pi t, cos 4 pi t] (SPEC.md:363 leaves
the embedding to the implementation); norm = RunningNorm::apply
(nn.cpp:272-277).  Mlp = 3 tanh hidden layers, flat parameters in the
nn.cpp:16-38 layout (W column-major).

Parity status: the reference's learner (learn.cpp) is absent, so there is no
reference binary for this path — "parity unpinned"; the restatement is pinned
by SPEC.md's sample_action examples (psi = 0 -> a = a0; psi = c -> a = a0 + c;
deterministic mode repeatable) and the Mlp init/forward pins of oracle.py.
"""
import numpy as np


def time_features(t):
    w = 2.0 * np.pi * t
    return np.array([t, np.sin(w), np.cos(w), np.sin(2 * w), np.cos(2 * w)])


def mlp_layers(theta, n_in, hidden, n_out):
    """[(W, b)] x 4 from the flat Mlp parameters (nn.cpp:16-27)."""
    dims = [(hidden, n_in), (hidden, hidden), (hidden, hidden), (n_out, hidden)]
    out, o = [], 0
    for r, c in dims:
        W = np.asarray(theta[o:o + r * c]).reshape(c, r).T  # column-major
        b = np.asarray(theta[o + r * c:o + r * c + r])
        out.append((W, b))
        o += r * c + r
    assert o == len(theta)
    return out


def mlp_forward(layers, x):
    h = x
    for W, b in layers[:3]:
        h = np.tanh(h @ W.T + b)
    W, b = layers[3]
    return h @ W.T + b


def running_norm_apply(x, mean, var, count):
    if count == 0:
        return x
    sd = np.maximum(np.sqrt(var + 1e-8), 1e-6)
    return (x - mean) / sd


def sample_action(pi_theta, log_std, psi_theta, obs, hidden, n_ode=20, dt=0.05, eps=None, norm=None,
                  head_scale=1.0, head_offset=0.0):
    """Returns (a, a0, logprob) per row of obs [n x D] (f64)."""
    obs = np.asarray(obs, dtype=np.float64)
    n, D = obs.shape
    nm = len(log_std)
    s = running_norm_apply(obs, *norm) if norm is not None else obs
    pi = mlp_layers(pi_theta, D, hidden, nm)
    psi = mlp_layers(psi_theta, 5 + D + nm, hidden, nm)
    mean = head_scale * mlp_forward(pi, s) + head_offset
    log_std = np.asarray(log_std, dtype=np.float64)
    if eps is None:
        a0 = mean
        logp = np.zeros(n)
    else:
        a0 = mean + np.exp(log_std) * eps
        logp = np.sum(-0.5 * eps * eps - log_std - 0.5 * np.log(2 * np.pi), axis=1)
    a = a0.copy()
    for k in range(n_ode):
        phi = np.broadcast_to(time_features(k * dt), (n, 5))
        a = a + mlp_forward(psi, np.concatenate([phi, s, a], axis=1)) * dt
    return a, a0, logp


def compute_gae(reward, done, value, bootstrap, gamma, lam):
    """compute_gae, [h x E] arrays, f64: returns (advantages, returns)."""
    reward, value = np.asarray(reward, np.float64), np.asarray(value, np.float64)
    nd = 1.0 - (np.asarray(done) & 1).astype(np.float64)
    h = reward.shape[0]
    adv = np.zeros_like(reward)
    next_v, next_a = np.asarray(bootstrap, np.float64), 0.0
    for t in range(h - 1, -1, -1):
        delta = reward[t] + gamma * next_v * nd[t] - value[t]
        next_a = delta + gamma * lam * nd[t] * next_a
        adv[t] = next_a
        next_v = value[t]
    return adv, adv + value


# ---- PPO minibatch shuffle (rollout.cu msk_rollout_minibatch) -------------
def _mix32(x):
    x = np.uint64(x) & np.uint64(0xFFFFFFFF)
    x ^= x >> np.uint64(16)
    x = (x * np.uint64(0x7FEB352D)) & np.uint64(0xFFFFFFFF)
    x ^= x >> np.uint64(15)
    x = (x * np.uint64(0x846CA68B)) & np.uint64(0xFFFFFFFF)
    x ^= x >> np.uint64(16)
    return int(x)


def minibatch_key(seed, epoch):
    """splitmix64 of (seed, epoch), as msk_rollout_minibatch."""
    M = (1 << 64) - 1
    z = (seed + 0x9E3779B97F4A7C15 * (epoch + 1)) & M
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    return z ^ (z >> 31)


def feistel_permutation(n, key):
    """The epoch shuffle: perm[i] for i < n (4-round Feistel on an even-bit
    domain >= n, cycle-walked into [0, n))."""
    bits = 2
    while (1 << bits) < n:
        bits += 2
    hb = bits // 2
    mask = (1 << hb) - 1
    out = np.empty(n, dtype=np.int64)
    for i in range(n):
        x = i
        while True:
            left, right = x >> hb, x & mask
            for rnd in range(4):
                k = ((key >> (16 * rnd)) ^ (0x9E3779B9 * (rnd + 1))) & 0xFFFFFFFF
                t = left ^ (_mix32(right ^ k) & mask)
                left, right = right, t
            x = (left << hb) | right
            if x < n:
                break
        out[i] = x
    return out
