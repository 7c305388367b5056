"""CPU tests of the parity oracle (oracle/msk_oracle.c).

The oracle is pinned three ways:
  1. SPEC.md known answers (the only golden numbers the reference documents,
     SPEC.md:38-76, 126-187, 245) and external KATs (std::mt19937_64);
  2. bit-exact agreement with the reference itself, compiled from
     /root/reference sources (oracle/_ref) — when that build is present;
  3. the committed golden fixtures tests/golden/*.npz, produced by the
     reference (tests/golden/make_golden.py), so (2) also holds where
     /root/reference does not exist.
"""
import math
import os

import numpy as np
import pytest

from conftest import model_paths
from golden_cases import CASES
from oracle import oracle as om
from oracle.ref import REF_SO, env_config

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")
HAVE_REF = os.path.exists(REF_SO)


@pytest.fixture(scope="module")
def L():
    return om.lib()


# ---- muscle.cpp known answers --------------------------------
def test_force_length_anchors(L):
    assert L.om_force_length_active(1.0) == 1.0
    assert abs(L.om_force_length_active(1.45) - math.exp(-1)) < 1e-15
    assert L.om_force_length_active(0.3) < 0.1


def test_force_velocity_anchors(L):
    assert L.om_force_velocity(0.0) == 1.0
    assert L.om_force_velocity(-1.0) == 0.0
    assert L.om_force_velocity(-3.0) == 0.0
    v2 = L.om_force_velocity(2.0)
    assert 1.0 < v2 <= 1.4 and abs(v2 - 1.3448275862069) < 1e-12
    grid = np.linspace(-1.5, 5, 2001)
    vals = np.array([L.om_force_velocity(v) for v in grid])
    assert np.all(np.diff(vals) >= 0)  # monotone


def test_force_passive_anchors(L):
    assert L.om_force_passive(1.0) == 0.0
    assert L.om_force_passive(0.8) == 0.0
    assert abs(L.om_force_passive(1.5) - 1.0) < 1e-15


def test_mtu_force_examples(L):
    assert L.om_mtu_force(1.0, 1.0, 0.0, 100.0) == 100.0
    assert L.om_mtu_force(0.0, 1.0, 0.0, 100.0) == 0.0
    assert abs(L.om_mtu_force(0.5, 1.2, -0.3, 100.0) - 45.9041272945895) < 1e-10


def test_activation_step_examples(L):
    assert abs(L.om_activation_step(0.0, 1.0, 0.002, 0.010, 0.040) - 0.3296799539643607) < 1e-6
    assert abs(L.om_activation_step(1.0, 0.0, 0.002, 0.010, 0.040) - 0.9048374180359595) < 1e-6
    assert L.om_activation_step(0.3, 0.3, 0.002, 0.010, 0.040) == 0.3


def test_activation_bounded_and_asymmetric(L):
    rng = np.random.default_rng(0)
    for _ in range(200):
        a = rng.uniform()
        for u in rng.uniform(size=50):
            a = L.om_activation_step(a, u, 0.002, 0.010, 0.040)
            assert 0.0 <= a <= 1.0
    # rise to 0.63 is faster than decay to 0.37
    a, n_up = 0.0, 0
    while a < 0.63:
        a = L.om_activation_step(a, 1.0, 0.002, 0.010, 0.040)
        n_up += 1
    a, n_dn = 1.0, 0
    while a > 0.37:
        a = L.om_activation_step(a, 0.0, 0.002, 0.010, 0.040)
        n_dn += 1
    assert n_up < n_dn


def test_wrap_angle(L):
    assert abs(L.om_wrap_angle(3.1 - (-3.1)) - (-0.08318530717958694)) < 1e-15
    assert L.om_wrap_angle(-math.pi) == math.pi  # (-pi, pi]


# ---- skeleton.cpp properties -------------------------------
@pytest.mark.parametrize("name", ["arm2_m6", "walker5_m16", "wb700"])
def test_mass_matrix_symmetric_pd(assets, name):
    m = om.OracleModel(model_paths(name)[0])
    rng = np.random.default_rng(1)
    for _ in range(30 if name != "wb700" else 3):
        q = rng.uniform(-1, 1, m.nq)
        M = m.mass_matrix(q)
        assert np.abs(M - M.T).max() < 1e-12
        assert np.linalg.eigvalsh(M).min() > 0


@pytest.mark.parametrize("name", ["arm2_m6", "walker5_m16"])
def test_moment_arms_match_finite_differences(assets, name):
    m = om.OracleModel(model_paths(name)[0])
    rng = np.random.default_rng(2)
    q = rng.uniform(-0.5, 0.5, m.nq)
    J = m.moment_arms(q)
    h = 1e-6
    for i in range(m.nm):
        for j in range(m.nq):
            qp, qm = q.copy(), q.copy()
            qp[j] += h
            qm[j] -= h
            fd = -(m.mtu_length(qp, i) - m.mtu_length(qm, i)) / (2 * h)
            assert abs(J[i, j] - fd) <= 1e-4 * max(abs(fd), 1e-3)


def test_pendulum_closed_forms(assets):
    m = om.OracleModel(model_paths("pendulum1_m2")[0])
    d = m.d
    mass, I, com = d["link_mass"][0], d["link_inertia"][0], d["link_com"][0]
    M = m.mass_matrix(np.array([0.3]))
    assert abs(M[0, 0] - (I + mass * com * com)) < 1e-14
    # horizontal (mount -pi/2, q = pi/2 -> link along +x): gravity torque m g d
    C = m.bias_forces(np.array([math.pi / 2]), np.array([0.0]))
    assert abs(C[0] - mass * 9.81 * com) < 1e-12
    # hanging straight down at rest: zero torque
    C0 = m.bias_forces(np.array([0.0]), np.array([0.0]))
    assert abs(C0[0]) < 1e-12


def test_two_link_fk_closed_form(assets):
    m = om.OracleModel(model_paths("arm2_m6")[0])
    q = np.array([0.4, 1.1])
    pos, ang = m.key_bodies(q)
    l0 = m.d["link_length"][0]
    c0, c1 = m.d["link_com"]
    a0 = -math.pi / 2 + q[0]
    a1 = a0 + q[1]
    p1 = np.array([l0 * math.cos(a0), l0 * math.sin(a0)]) + c1 * np.array([math.cos(a1), math.sin(a1)])
    assert np.abs(pos[1] - p1).max() < 1e-14
    assert abs(ang[1] - a1) < 1e-15


def test_passive_pendulum_energy_drift(assets, tmp_path):
    """Passive, undamped, contact-free chain conserves energy within 2% over 10 s."""
    import json

    path = model_paths("pendulum1_m2")[0]
    js = json.load(open(path))
    js["joints"][0]["damping"] = 0.0
    js["joints"][0]["limits"] = [-100.0, 100.0]
    for mu in js["muscles"]:  # no passive stretch: keep fibres slack
        mu["tendon_slack"] = 10.0
    p = tmp_path / "pend.json"
    p.write_text(json.dumps(js))
    m = om.OracleModel(str(p))
    q, dq = np.array([math.pi / 2]), np.array([0.0])
    e0 = m.mechanical_energy(q, dq)
    act = np.zeros(m.nm)
    lm = np.full(m.nm, 0.01)
    vm, fm = np.zeros(m.nm), np.zeros(m.nm)
    u = np.zeros(m.nm)
    s = dict(q=q, dq=dq, act=act, l_m=lm, v_m=vm, f_m=fm)
    worst = 0.0
    # released from horizontal: energy scale = m g d (the swing's KE at the bottom)
    scale = m.d["link_mass"][0] * 9.81 * m.d["link_com"][0]
    for _ in range(5000):
        s, _, bad = m.substep(s["q"], s["dq"], s["act"], s["l_m"], s["v_m"], s["f_m"], u)
        assert not bad
        worst = max(worst, abs(m.mechanical_energy(s["q"], s["dq"]) - e0) / scale)
    assert worst < 0.02


# ---- rng.hpp: std::mt19937_64 known answers ----------------------------------
def test_mt19937_64_known_answers(L):
    import ctypes as C

    e = om.OmEnv()
    L.om_rng_seed(C.byref(e), 5489)
    for _ in range(9999):
        L.om_rng_raw(C.byref(e))
    assert L.om_rng_raw(C.byref(e)) == 9981545732273789042  # C++ [rand.predef]
    L.om_rng_seed(C.byref(e), 12345)
    x = L.om_rng_raw(C.byref(e))
    assert x == 6597103971274460346
    assert (x >> 11) * 2.0 ** -53 == 0.35762972288842587


def test_philox_excitations_known_values():
    # Random123 Philox4x32-10 KAT: counter/key all zero -> 6627e8d5 e169c58d bc57ac4c 9b00dbd8
    L = om.lib()
    vals = [L.om_excitation(0, 0, 0, k) for k in range(4)]
    expect = [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    assert vals == [(x >> 8) / 16777216.0 for x in expect]


# ---- oracle vs reference ------------------------------------------------------
def _run_pair(name, n, steps, cfg_kw, mode=0):
    from oracle.ref import RefBatch, excitations

    mp, cp = model_paths(name)
    r = RefBatch(mp, cp, n, cfg=env_config(**cfg_kw), reward_mode=mode)
    o = om.OracleBatch(mp, cp, n, cfg=env_config(**cfg_kw), reward_mode=mode)
    ob1, f1 = r.reset()
    ob2, f2 = o.reset()
    assert (f1 == f2).all() and np.array_equal(ob1, ob2)
    for s in range(steps):
        a = excitations(99, s, n, r.nm)
        x, y = r.step(a), o.step(a)
        for k in x:
            assert np.array_equal(x[k], y[k]), (name, s, k)
        d = (x["flags"] & 1).astype(np.uint8)
        if d.any():
            r.record_own_outcomes()
            o.record_own_outcomes()
            _, fa = r.reset(mask=d)
            _, fb = o.reset(mask=d)
            assert np.array_equal(fa, fb)
    for k, v in r.get_state().items():
        assert np.array_equal(v, o.get_state()[k]), k
    assert np.array_equal(r.get_sampler(), o.get_sampler())


@pytest.mark.skipif(not HAVE_REF, reason="reference build oracle/_ref absent")
@pytest.mark.parametrize("name,n,steps,cfg_kw,mode", [
    ("pendulum1_m2", 3, 60, dict(episode_horizon=20), 0),
    ("arm2_m6", 4, 80, dict(episode_horizon=25), 2),
    ("walker5_m16", 4, 40, dict(episode_horizon=1000, termination_body_err=0.3), 0),
    ("wb700", 2, 2, dict(episode_horizon=1000), 2),
    ("arm2_m6", 1, 1000, dict(episode_horizon=1000, rsi=False), 0),  # BASELINE c1: 1 env, 1000 steps
])
def test_oracle_bit_exact_vs_reference(assets, name, n, steps, cfg_kw, mode):
    _run_pair(name, n, steps, cfg_kw, mode)


# ---- oracle vs golden fixtures (made by the reference) -----------------------
GOLDEN_CASES = sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz") and f[:-4] in CASES) if os.path.isdir(GOLDEN) else []


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_oracle_reproduces_reference_golden(assets, name):
    g = np.load(os.path.join(GOLDEN, name + ".npz"))
    n, steps, mode = [int(x) for x in g["meta"]]
    cfg_kw = CASES[name][2]
    mp, cp = model_paths(name)
    o = om.OracleBatch(mp, cp, n, cfg=env_config(**cfg_kw), reward_mode=mode)
    o.set_sampler(g["ema0"])
    obs0, fr0 = o.reset()
    assert np.array_equal(fr0, g["frames0"])
    assert np.array_equal(obs0, g["obs0"])
    for s in range(steps):
        r = o.step(g["actions"][s])
        assert np.array_equal(r["flags"], g["flags"][s])
        for k in ("delta", "obs", "reward_aux", "power"):
            assert np.array_equal(r[k], g[k][s]), (s, k)
        st = o.get_state()
        for k in ("q", "dq", "act", "l_m", "v_m", "f_m", "t", "ints"):
            assert np.array_equal(st[k], g["state_" + k][s]), (s, k)
        d = (r["flags"] & 1).astype(np.uint8)
        if d.any():
            o.record_own_outcomes()
            _, f = o.reset(mask=d)
            assert np.array_equal(np.where(d > 0, f, -1), g["reset_frames"][s])
    assert np.array_equal(o.get_sampler(), g["ema_end"])
    assert np.array_equal(o.rng_raw(0, 400), g["rng_draws"])


# ---- discriminator (nn.cpp Mlp + SPEC reward_from_discriminator) -------------
def test_mlp_init_matches_reference_rng_golden():
    """Mlp(shape, seed 7) weights from the reference's own Rng stream (golden)."""
    g = np.load(os.path.join(GOLDEN, "mlp_seed7.npz"))
    assert np.array_equal(om.mlp_init(9, 16, 7), g["small"])
    big = om.mlp_init(102, 256, 7)
    assert big.size == int(g["big_len"][0]) == om.mlp_param_count(102, 256)
    assert np.array_equal(big[:512], g["big_head"]) and np.array_equal(big[-512:], g["big_tail"])
    assert np.sum(big) == g["big_sum"][0]


@pytest.mark.skipif(not HAVE_REF, reason="reference build (oracle/_ref) absent")
def test_mlp_init_matches_reference_rng_live():
    from oracle.ref import rng_uniform

    theta = om.mlp_init(9, 16, 3)
    u = rng_uniform(3, 0.0, 1.0, 16 * 9)
    s = 1.0 / math.sqrt(9.0)
    assert np.array_equal(theta[:16 * 9], -s + (s - -s) * u)


def test_discriminator_spec_examples():
    """zero-initialised head -> D = 0.5 -> r = log 2; clamp
    bounds -> r in (1e-4, 9.2103]; r monotone in D."""
    th = om.mlp_init(9, 16, 7, final_init_scale=0.0)
    x = np.random.default_rng(0).normal(0, 1, (5, 9))
    assert np.allclose(om.mlp_forward_sigmoid(th, 9, 16, x), 0.5, atol=0, rtol=0)
    assert np.allclose(om.disc_reward(th, 9, 16, x), math.log(2.0), rtol=0, atol=1e-15)
    L = om.lib()
    assert abs(L.om_disc_reward(1.0) - 9.2103) < 1e-4 and abs(L.om_disc_reward(0.0) - 1.00005e-4) < 1e-8
    d = np.linspace(0, 1, 101)
    r = np.array([L.om_disc_reward(v) for v in d])
    assert np.all(np.diff(r) >= 0)


def test_mlp_forward_matches_numpy():
    """Independent matrix-arithmetic evaluation (SPEC.md nn forward example)."""
    n_in, h = 7, 16
    th = om.mlp_init(n_in, h, 11)
    x = np.random.default_rng(1).normal(0, 0.5, (6, n_in))
    o, ws = 0, []
    for r, c in [(h, n_in), (h, h), (h, h), (1, h)]:
        W = th[o:o + r * c].reshape(c, r).T  # column-major
        b = th[o + r * c:o + r * c + r]
        ws.append((W, b))
        o += r * c + r
    a = x
    for W, b in ws[:3]:
        a = np.tanh(a @ W.T + b)
    z = a @ ws[3][0].T + ws[3][1]
    assert np.allclose(om.mlp_forward_sigmoid(th, n_in, h, x), 1 / (1 + np.exp(-z[:, 0])), rtol=1e-13, atol=0)


# ---- RNG checkpoint state (Env::rng(), Rng::serialize; env.hpp:120, rng.hpp:56-68) ----
def test_oracle_rng_state_matches_reference_serialize_golden(assets):
    """The oracle's mt19937_64 engine state, written in Rng::serialize's format,
    equals the reference's own serialize() text at construction and after every
    RSI reset round (tests/golden/rng_serialize.json, made by oracle/_ref)."""
    import json

    g = json.load(open(os.path.join(GOLDEN, "rng_serialize.json")))
    c = g["case"]
    mp, cp = model_paths(c["model"])
    o = om.OracleBatch(mp, cp, c["n"], cfg=env_config(**c["cfg"]))
    o.set_sampler(np.tile(np.array(g["ema"]), (c["n"], 1)))
    assert [o.rng_serialize(e) for e in range(c["n"])] == g["serialize"][0]
    for r in range(c["rounds"]):
        _, f = o.reset()
        assert f.tolist() == g["frames"][r]
        assert [o.rng_serialize(e) for e in range(c["n"])] == g["serialize"][r + 1]


@pytest.mark.skipif(not HAVE_REF, reason="reference build oracle/_ref absent")
def test_reference_rng_deserialize_restores_the_reset_sequence(assets):
    """Rng::deserialize of a saved serialize() replays the same start frames
    (the checkpoint contract the device's get/set_rng mirrors)."""
    from oracle.ref import RefBatch

    mp, cp = model_paths("arm2_m6")
    b = RefBatch(mp, cp, 2, cfg=env_config(episode_horizon=30, rsi=True))
    b.reset()
    saved = [b.rng_serialize(e) for e in range(2)]
    first = [b.reset()[1].tolist() for _ in range(4)]
    for e in range(2):
        b.rng_deserialize(e, saved[e])
    assert [b.reset()[1].tolist() for _ in range(4)] == first


@pytest.mark.skipif(not HAVE_REF, reason="reference build oracle/_ref absent")
def test_discriminator_and_policy_mlps_match_reference_nn_cpp():
    """The reward oracle's Mlp (om_mlp_forward_sigmoid, the D(Δ) of every GPU reward
    test) and the policy oracle's Mlp (oracle/policy.py, Head::Affine) equal the
    reference's own Mlp::forward (nn.cpp:54-73) to f64 rounding."""
    from oracle.policy import mlp_forward, mlp_layers
    from oracle.ref import HEAD_AFFINE, ref_mlp_forward

    rng = np.random.default_rng(4)
    for din, H in ((9, 16), (102, 256)):
        th = om.mlp_init(din, H, 7) + rng.normal(0, 0.02, om.mlp_param_count(din, H))
        X = rng.normal(0, 1.0, (11, din))
        ref = ref_mlp_forward(th, din, H, 1, X)[:, 0]
        assert np.max(np.abs(om.mlp_forward_sigmoid(th, din, H, X) - ref)) <= 1e-14
        r_ref = -np.log(1.0 - np.clip(ref, 1e-4, 1.0 - 1e-4))
        assert np.max(np.abs(om.disc_reward(th, din, H, X) - r_ref)) <= 1e-13
    th = om.mlp_init(40, 64, 3, n_out=24)
    X = rng.normal(0, 1.0, (9, 40))
    y = 0.5 * mlp_forward(mlp_layers(th, 40, 64, 24), X) + 0.25
    ref = ref_mlp_forward(th, 40, 64, 24, X, head=HEAD_AFFINE, affine=(0.5, 0.25))
    assert np.max(np.abs(y - ref)) <= 1e-13 * max(1.0, np.abs(ref).max())


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="reference build oracle/_ref absent")
def test_reference_bench_with_discriminator_reward():
    """The CPU arm's c4 tracking reward: the reference's own Mlp (Head::Sigmoid) as
    Env::step's TrackingRewardFn; a wrong parameter count is refused."""
    from oracle.oracle import mlp_init
    from oracle.ref import RefBatch, env_config

    mp, cp = model_paths("arm2_m6")
    b = RefBatch(mp, cp, 2, cfg=env_config(episode_horizon=50, rsi=True), threads=1)
    with pytest.raises(ValueError):
        b.set_discriminator(np.zeros(5), 16)
    b.set_discriminator(mlp_init(b.delta_dim, 16, 7), 16)
    b.reset()
    secs, steps = b.bench(3)
    assert steps == 6 and secs > 0
