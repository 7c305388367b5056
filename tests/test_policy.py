"""On-device policy sampling vs the f64 oracle (oracle/policy.py).

Tolerances (bf16 tensor-core operands, fp32 accumulation):
  one GEMM layer  vs torch fp32 on the same bf16-rounded operands: rel 1e-4 (linear), 4e-3 abs (tanh -> bf16)
  full sample (π⁽⁰⁾ + 20 flow steps) vs f64: |Δa| <= 2e-2 (measured ~5e-3, tools/policy_check.py)
  SPEC.md:391-393 examples: ψ ≡ 0 -> a = a⁽⁰⁾ exactly; ψ ≡ c -> a = a⁽⁰⁾ + c (1e-5); deterministic repeatable.
"""
import numpy as np
import pytest

from oracle.oracle import mlp_init
from oracle.policy import sample_action

pytestmark = pytest.mark.gpu

D, NM, H = 40, 24, 64


def _bf16(x):
    import torch

    return torch.as_tensor(np.asarray(x, dtype=np.float32)).to(torch.bfloat16).float()


@pytest.mark.parametrize("epi", [0, 1])
def test_tiled_gemm_matches_torch(epi):
    import ctypes as C

    import torch

    import paper_2603_29332_b200 as pk

    rng = np.random.default_rng(epi)
    M, K, N = 300, 200, 300  # ragged in every dimension, two N tiles
    X = rng.normal(0, 1, (M, K)).astype(np.float32)
    W = rng.normal(0, 1 / np.sqrt(K), (N, K))
    b = rng.normal(0, 0.1, N).astype(np.float32)
    Wc = np.asfortranarray(W).ravel(order="F")  # column-major, as Mlp stores it
    Y = np.zeros((M, N), dtype=np.float32)
    rc = pk.lib().msk_gemm_test(X.ctypes.data, M, K, Wc.ctypes.data, b.ctypes.data, N, epi, Y.ctypes.data)
    assert rc == 0
    ref = (_bf16(X) @ _bf16(W).T + torch.as_tensor(b)).numpy()
    if epi == 1:
        assert np.abs(Y - ref).max() <= 1e-4 * max(1.0, np.abs(ref).max())
    else:
        assert np.abs(Y - np.tanh(ref)).max() <= 4e-3


def _params(seed, psi_scale=0.3):
    pi = mlp_init(D, H, seed, n_out=NM)
    psi = mlp_init(5 + D + NM, H, seed + 1, n_out=NM, final_init_scale=psi_scale)
    log_std = np.full(NM, -1.0)  # SPEC.md:372 init log-std
    return pi, log_std, psi


def _policy(pi, log_std, psi, **kw):
    import paper_2603_29332_b200 as pk

    return pk.Policy(D, NM, H, pi, log_std, psi, max_envs=512, **kw)


def test_policy_deterministic_matches_oracle():
    import torch

    pi, ls, psi = _params(3)
    p = _policy(pi, ls, psi, head_scale=0.5, head_offset=0.5)
    rng = np.random.default_rng(0)
    obs = rng.normal(0, 1, (200, D)).astype(np.float32)
    mean, var = rng.normal(0, 0.2, D), rng.uniform(0.5, 2.0, D)
    p.set_norm(mean, var, 100.0)
    a = p.sample(torch.as_tensor(obs, device="cuda")).cpu().numpy()
    ref, _, _ = sample_action(pi, ls, psi, obs, H, norm=(mean, var, 100.0), head_scale=0.5, head_offset=0.5)
    err = np.abs(a - ref).max()
    assert err <= 2e-2, err
    # deterministic mode is repeatable, and the CUDA-graph replay is identical
    b = p.sample(torch.as_tensor(obs, device="cuda")).cpu().numpy()
    g = p.sample(torch.as_tensor(obs, device="cuda"), graph=True).cpu().numpy()
    g2 = p.sample(torch.as_tensor(obs, device="cuda"), graph=True).cpu().numpy()
    assert np.array_equal(a, b) and np.array_equal(a, g) and np.array_equal(g, g2)
    p.close()


def test_graph_replay_follows_normaliser_changes():
    """A graph captured before msk_policy_set_norm must apply the new statistics
    (the normaliser is part of every replay, not of the capture key)."""
    import torch

    pi, ls, psi = _params(4)
    p = _policy(pi, ls, psi)
    rng = np.random.default_rng(5)
    obs = torch.as_tensor(rng.normal(0, 1, (150, D)).astype(np.float32), device="cuda")
    g0 = p.sample(obs, graph=True).clone()  # count 0: identity normaliser
    e0 = p.sample(obs).clone()
    assert torch.equal(g0, e0)
    mean, var = rng.normal(0, 0.5, D), rng.uniform(0.2, 3.0, D)
    p.set_norm(mean, var, 50.0)
    g1 = p.sample(obs, graph=True).clone()
    e1 = p.sample(obs).clone()
    assert torch.equal(g1, e1)
    assert not torch.equal(g0, g1)
    ref, _, _ = sample_action(pi, ls, psi, obs.cpu().numpy(), H, norm=(mean, var, 50.0))
    assert np.abs(g1.cpu().numpy() - ref).max() <= 2e-2
    p.set_norm(None, None, 0.0)  # back to the identity
    g2 = p.sample(obs, graph=True).clone()
    assert torch.equal(g2, g0)
    p.close()


def test_policy_spec_examples():
    """ψ ≡ 0 -> a = a⁽⁰⁾; ψ ≡ c -> a = a⁽⁰⁾ + c."""
    import torch

    pi, ls, psi = _params(5)
    zero = np.zeros_like(psi)
    p = _policy(pi, ls, zero)
    obs = torch.as_tensor(np.random.default_rng(1).normal(0, 1, (130, D)).astype(np.float32), device="cuda")
    a0 = torch.empty(130, NM, device="cuda")
    a = p.sample(obs, a0=a0)
    assert torch.equal(a, a0)
    p.close()
    const = zero.copy()
    c = np.linspace(-0.3, 0.4, NM)
    const[-NM:] = c  # ψ head bias only
    p = _policy(pi, ls, const)
    a = p.sample(obs, a0=a0)
    assert np.abs((a - a0).cpu().numpy() - c).max() <= 1e-5
    p.close()


def test_policy_explore_noise_and_logprob():
    import torch

    pi, ls, psi = _params(7)
    p = _policy(pi, ls, np.zeros_like(psi))
    n = 500
    obs = torch.as_tensor(np.random.default_rng(2).normal(0, 1, (n, D)).astype(np.float32), device="cuda")
    mean = p.sample(obs).clone()
    a0 = torch.empty(n, NM, device="cuda")
    lp = torch.empty(n, device="cuda")
    a = p.sample(obs, explore=True, seed=11, step=3, a0=a0, logprob=lp)
    eps = ((a0 - mean) / np.exp(-1.0)).cpu().numpy()
    assert abs(eps.mean()) < 0.05 and abs(eps.std() - 1.0) < 0.05
    ref_lp = np.sum(-0.5 * eps * eps + 1.0 - 0.5 * np.log(2 * np.pi), axis=1)
    assert np.abs(lp.cpu().numpy() - ref_lp).max() <= 1e-3 * np.abs(ref_lp).max()
    assert torch.equal(a, a0)  # ψ ≡ 0
    # same (seed, step, env) -> same noise; another step -> different noise
    a0b = torch.empty_like(a0)
    p.sample(obs, explore=True, seed=11, step=3, a0=a0b)
    assert torch.equal(a0, a0b)
    p.sample(obs, explore=True, seed=11, step=4, a0=a0b)
    assert not torch.equal(a0, a0b)
    p.close()


def test_rollout_gae_matches_oracle_and_spec():
    """On-device GAE vs the f64 recursion; SPEC examples."""
    import torch

    import paper_2603_29332_b200 as pk
    from oracle.policy import compute_gae

    E, h = 300, 8
    rng = np.random.default_rng(4)
    r = rng.normal(0, 1, (h, E)).astype(np.float32)
    v = rng.normal(0, 1, (h, E)).astype(np.float32)
    boot = rng.normal(0, 1, E).astype(np.float32)
    flags = (rng.uniform(0, 1, (h, E)) < 0.2).astype(np.uint8)  # bit 0 = done
    ro = pk.Rollout(E, h, 3, 2, 1)
    for t in range(h):
        ro.record(t, reward=torch.as_tensor(r[t], device="cuda"), flags=torch.as_tensor(flags[t], device="cuda"),
                  value=torch.as_tensor(v[t], device="cuda"))
    bt = torch.as_tensor(boot, device="cuda")
    adv, ret = ro.gae(bt, gamma=0.99, lam=0.95, normalize=False)
    a_ref, r_ref = compute_gae(r, flags, v, boot, 0.99, 0.95)
    assert np.abs(adv.cpu().numpy() - a_ref).max() <= 1e-4 * max(1.0, np.abs(a_ref).max())
    assert np.abs(ret.cpu().numpy() - r_ref).max() <= 1e-4 * max(1.0, np.abs(r_ref).max())
    # normalised advantages: zero mean, unit variance over the batch
    adv_n, _ = ro.gae(bt, gamma=0.99, lam=0.95, normalize=True)
    an = adv_n.cpu().numpy().astype(np.float64)
    assert abs(an.mean()) < 1e-5 and abs(an.std() - 1.0) < 1e-4
    # lambda = 0 -> TD residual; single done step -> A = r - V
    adv0, _ = ro.gae(bt, gamma=0.99, lam=0.0, normalize=False)
    nxt = np.concatenate([v[1:], boot[None]], 0)
    td = r + 0.99 * nxt * (1 - (flags & 1)) - v
    assert np.abs(adv0.cpu().numpy() - td).max() <= 1e-5
    d = (flags[-1] & 1) == 1
    assert np.abs(adv0.cpu().numpy()[-1][d] - (r[-1] - v[-1])[d]).max() <= 1e-6
    ro.close()


def test_rollout_minibatches_are_a_keyed_permutation():
    """PPO minibatching (msk_rollout_minibatch): every epoch's minibatches
    partition the h*E records (a permutation equal to the oracle's Feistel
    shuffle, deterministic in (seed, epoch), different across epochs) and
    gather exactly the stored rows and the last GAE's advantages / returns."""
    import torch

    import paper_2603_29332_b200 as pk
    from oracle.policy import feistel_permutation, minibatch_key

    E, h, D, NA = 37, 8, 12, 5  # 296 records, ragged last minibatch
    ro = pk.Rollout(E, h, D, NA, 1)
    rng = np.random.default_rng(8)
    obs = rng.normal(0, 1, (h, E, D)).astype(np.float32)
    act = rng.normal(0, 1, (h, E, NA)).astype(np.float32)
    rew = rng.normal(0, 1, (h, E)).astype(np.float32)
    val = rng.normal(0, 1, (h, E)).astype(np.float32)
    for t in range(h):
        ro.record(t, obs=torch.as_tensor(obs[t], device="cuda"), a0=torch.as_tensor(act[t] * 2, device="cuda"),
                  actions=torch.as_tensor(act[t], device="cuda"), logprob=torch.as_tensor(rew[t] * 3, device="cuda"),
                  reward=torch.as_tensor(rew[t], device="cuda"),
                  flags=torch.zeros(E, dtype=torch.uint8, device="cuda"), value=torch.as_tensor(val[t], device="cuda"))
    adv, ret = ro.gae(torch.zeros(E, device="cuda"), normalize=True)
    adv, ret = adv.cpu().numpy().reshape(-1), ret.cpu().numpy().reshape(-1)
    n, mb = h * E, 50
    orders = []
    for epoch in (0, 1):
        ids = []
        for b in range((n + mb - 1) // mb):
            out = {k: v.cpu().numpy() for k, v in ro.minibatch(11, epoch, b, mb, D, NA).items()}
            i = out["record_ids"].astype(np.int64)
            ids.append(i)
            assert np.array_equal(out["obs"], obs.reshape(n, D)[i])
            assert np.array_equal(out["actions"], act.reshape(n, NA)[i])
            assert np.array_equal(out["a0"], 2 * act.reshape(n, NA)[i])
            assert np.array_equal(out["logprob"], 3 * rew.reshape(n)[i])
            assert np.array_equal(out["value"], val.reshape(n)[i])
            assert np.array_equal(out["advantages"], adv[i]) and np.array_equal(out["returns"], ret[i])
        order = np.concatenate(ids)
        assert np.array_equal(np.sort(order), np.arange(n))
        assert np.array_equal(order, feistel_permutation(n, minibatch_key(11, epoch)))
        orders.append(order)
    assert not np.array_equal(orders[0], orders[1])
    again = ro.minibatch(11, 1, 0, mb, D, NA)["record_ids"].cpu().numpy()
    assert np.array_equal(again, orders[1][:mb])
    ro.close()


_PAIR_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2603_29332_b200 as pk
rng = np.random.default_rng(5)
M, K, N = 512, 320, 512   # 4 row tiles: CTA pairs apply; two N tiles, ragged K
X = rng.normal(0, 1, (M, K)).astype(np.float32)
W = rng.normal(0, 1 / np.sqrt(K), (N, K))
b = rng.normal(0, 0.1, N).astype(np.float32)
Wc = np.asfortranarray(W).ravel(order="F")
for epi in (0, 1):
    Y = np.zeros((M, N), dtype=np.float32)
    assert pk.lib().msk_gemm_test(X.ctypes.data, M, K, Wc.ctypes.data, b.ctypes.data, N, epi, Y.ctypes.data) == 0
    np.save(sys.argv[2] + f"_{epi}.npy", Y)
"""


def test_cta_pair_gemm_equals_single_cta(tmp_path):
    """The opt-in CTA-pair GEMM (MSK_GEMM_2CTA: tcgen05.mma.cta_group::2, both CTAs'
    TMA tensor copies completing on the leader's barrier) gives the single-CTA
    kernel's results bit for bit (same K-order per output element)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for mode, env in (("single", {}), ("pair", {"MSK_GEMM_2CTA": "1"})):
        base = str(tmp_path / mode)
        r = subprocess.run([sys.executable, "-c", _PAIR_SCRIPT, root, base], env={**os.environ, **env},
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs[mode] = [np.load(base + f"_{epi}.npy") for epi in (0, 1)]
    for a, b in zip(outs["single"], outs["pair"]):
        assert np.array_equal(a, b)


def test_persistent_ode_kernel_equals_per_layer_launches():
    """The opt-in persistent ψ-ODE kernel (MSK_POLICY_ODE=1: all hidden layers of the
    flow ODE in one launch, cluster-wide layer barriers over DSMEM) samples the same
    actions as the per-layer GEMM launches, bit for bit."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
import paper_2603_29332_b200 as pk
from test_policy import _params, D, NM, H
pi, ls, psi = _params(3)
p = pk.Policy(D, NM, H, pi, ls, psi, max_envs=512)
obs = torch.as_tensor(np.random.default_rng(2).normal(0, 1, (300, D)).astype(np.float32), device="cuda")
a = p.sample(obs, explore=True, seed=5, step=1)
np.save(sys.argv[2], a.cpu().numpy())
"""
    outs = []
    for env in ({}, {"MSK_POLICY_ODE": "1"}):
        path = os.path.join(str(os.environ.get("TMPDIR", "/tmp")), f"ode_{len(outs)}_{os.getpid()}.npy")
        r = subprocess.run([sys.executable, "-c", script, root, path], env={**os.environ, **env},
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(path))
    assert np.array_equal(outs[0], outs[1])
