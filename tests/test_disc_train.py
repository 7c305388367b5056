"""Discriminator training step — oracle pins
on CPU, device step vs the f64 oracle on the GPU.

Oracle (oracle/disc_train.py) pins: finite-difference gradient checks of the
loss (rel < 1e-5), the penalty equals ||dD/dΔ||², SPEC.md:419-420's
examples, the SPEC.md:418 training example, Adam's non-finite skip (nn.cpp:229-232).

Device tolerances (tests marked gpu), gradient norm-wise per parameter block:
  weight blocks (W0, W1, W2, w4; floor 1e-2 of the whole gradient's norm):
    math 0 (fp32-class split-bf16): rel 1e-4; math 1 (bf16): rel 5e-2
  bias blocks (b0, b1, b2, b4): column sums over the rows in which the D(0) row
  cancels most of the Δ rows (|Σ_r| is 60-1000x below Σ_r |.|), so their error
  is measured against the sum's condition ||Σ_r |row|||  (oracle
  bias_adjoint_rows): math 0 1e-5, math 1 5e-3
  loss: rel 1e-5 (math 0), 1e-3 (math 1)
  θ after 3 Adam steps: ||θ_gpu − θ_ref|| ≤ 1e-2 ||θ_ref − θ_0||
  published reward discriminator: as the bf16 reward path, 3e-3 max(1, |r|)
"""
import ctypes as C

import numpy as np
import pytest

from oracle.disc_train import Adam, disc_loss_grad, gradient_penalty_backward, mlp_forward_cache, train_discriminator
from oracle.oracle import disc_reward, mlp_init


def _fd_check(theta, din, H, delta, lam, idx, eps=1e-6):
    g = disc_loss_grad(theta, din, H, delta, lam)[3]
    worst = 0.0
    for i in idx:
        tp, tm = theta.copy(), theta.copy()
        tp[i] += eps
        tm[i] -= eps
        fd = (disc_loss_grad(tp, din, H, delta, lam)[0] - disc_loss_grad(tm, din, H, delta, lam)[0]) / (2 * eps)
        worst = max(worst, abs(fd - g[i]) / max(1e-6, abs(fd) + abs(g[i])))
    return worst


@pytest.mark.parametrize("lam", [0.0, 10.0])
def test_oracle_gradient_matches_finite_differences(lam):
    din, H = 7, 16
    theta = mlp_init(din, H, 7)
    rng = np.random.default_rng(1)
    delta = rng.normal(0, 0.5, (6, din))
    idx = rng.choice(len(theta), 60, replace=False)
    assert _fd_check(theta, din, H, delta, lam, idx) < 1e-5


def test_oracle_penalty_is_squared_input_gradient():
    din, H = 5, 16
    theta = mlp_init(din, H, 3)
    x = np.random.default_rng(2).normal(0, 1, (4, din))
    pen = gradient_penalty_backward(mlp_forward_cache(theta, din, H, x), np.zeros(len(theta)), din, H)
    eps, gx = 1e-6, np.zeros_like(x)
    for j in range(din):
        xp, xm = x.copy(), x.copy()
        xp[:, j] += eps
        xm[:, j] -= eps
        gx[:, j] = (mlp_forward_cache(theta, din, H, xp)["y"][:, 0] - mlp_forward_cache(theta, din, H, xm)["y"][:, 0]) / (2 * eps)
    assert np.allclose(pen, (gx ** 2).sum(1), rtol=1e-7)


def test_oracle_spec_examples():
    """zero-initialised head -> D = 0.5 everywhere, loss = 2 log 2
    (penalty 0: the input gradient vanishes with w4 = 0); λ = 0 -> pure logistic terms."""
    din, H = 9, 32
    th0 = mlp_init(din, H, 7, final_init_scale=0.0)
    delta = np.random.default_rng(3).normal(0, 1, (16, din))
    loss, logistic, pen, _ = disc_loss_grad(th0, din, H, delta, 10.0)
    assert abs(loss - 2 * np.log(2)) < 1e-14 and pen == 0.0
    th = mlp_init(din, H, 7)
    l0, lg0, p0, _ = disc_loss_grad(th, din, H, delta, 0.0)
    assert l0 == lg0 and p0 == 0.0
    l1, lg1, p1, _ = disc_loss_grad(th, din, H, delta, 10.0)
    assert lg1 == lg0 and abs(l1 - (lg1 + 10.0 * p1)) < 1e-14 and p1 > 0


def test_oracle_training_separates_zero_from_large_delta():
    """after training on a batch with large ||Δ||, D(0) > D(Δ_typical)."""
    din, H = 6, 16
    theta = mlp_init(din, H, 11)
    rng = np.random.default_rng(4)
    delta = rng.normal(0, 2.0, (64, din))
    adam = Adam(len(theta), 1e-2)
    for _ in range(60):
        train_discriminator(theta, din, H, delta, 10.0, adam)
    c0 = mlp_forward_cache(theta, din, H, np.zeros((1, din)))["y"][0, 0]
    cd = mlp_forward_cache(theta, din, H, delta)["y"][:, 0]
    assert adam.step_count == 60 and c0 > np.median(cd)


def test_oracle_adam_skips_non_finite_gradient():
    th = np.ones(4)
    a = Adam(4, 0.1)
    assert not a.step(th, np.array([1.0, np.nan, 0.0, 0.0]))
    assert a.skipped == 1 and a.step_count == 0 and np.all(th == 1.0)
    assert a.step(th, np.array([1.0, -1.0, 0.0, 2.0]))
    # first Adam step moves each parameter by lr * sign(g) (bias-corrected m / sqrt(v))
    assert np.allclose(th, [0.9, 1.1, 1.0, 0.9], atol=1e-7)


def test_trainer_entry_points_fail_cleanly():
    """Bad shapes -> status 1 before any device work; without a GPU -> status 3, no CPU fallback."""
    import paper_2603_29332_b200 as pk

    L = pk.lib()
    h = C.c_void_p()
    th = np.zeros(10)
    rc = L.msk_disc_trainer_create(5, 16, th.ctypes.data, th.size, 1e-3, 10.0, 64, 1, 0, C.byref(h))
    assert rc == 1 and not h.value and b"parameter count" in L.msk_disc_trainer_last_error(None)
    th = mlp_init(5, 16, 7)
    rc = L.msk_disc_trainer_create(5, 16, th.ctypes.data, th.size, 1e-3, 10.0, 64, 7, 0, C.byref(h))
    assert rc == 1 and b"math" in L.msk_disc_trainer_last_error(None)
    assert L.msk_disc_train_step(None, None, 1, 5, None, None) == 1
    import torch

    if not torch.cuda.is_available():
        rc = L.msk_disc_trainer_create(5, 16, th.ctypes.data, th.size, 1e-3, 10.0, 64, 1, 0, C.byref(h))
        assert rc == 3 and not h.value


# ---------------------------------------------------------------- GPU ----
def _blocks(din, H):
    o, out = 0, []
    for r, c in [(H, din), (H, H), (H, H), (1, H)]:
        out.append((o, o + r * c))
        out.append((o + r * c, o + r * c + r))
        o += r * c + r
    return out


def _block_rel(g, ref, din, H):
    """Worst weight-block error relative to max(||block||, 1e-2 ||grad||)."""
    floor = 1e-2 * np.linalg.norm(ref)
    return max(np.linalg.norm(g[a:b] - ref[a:b]) / max(np.linalg.norm(ref[a:b]), floor)
               for a, b in _blocks(din, H)[0::2])


def _bias_cond_rel(g, ref, theta, din, H, delta, lam):
    """Worst bias-block error relative to the condition of its column sum, ||Σ_r |row|||."""
    from oracle.disc_train import bias_adjoint_rows

    rows = bias_adjoint_rows(theta, din, H, delta, lam)
    return max(np.linalg.norm(g[a:b] - ref[a:b]) / np.linalg.norm(np.abs(rw).sum(0))
               for (a, b), rw in zip(_blocks(din, H)[1::2], rows))


@pytest.mark.gpu
@pytest.mark.parametrize("math,tol_g,tol_c,tol_l", [(0, 1e-4, 1e-5, 1e-5), (1, 5e-2, 5e-3, 1e-3)])
@pytest.mark.parametrize("din,H,B", [(9, 16, 37), (102, 256, 1000), (130, 200, 333)])
def test_device_gradient_matches_oracle(math, tol_g, tol_c, tol_l, din, H, B):
    import torch

    import paper_2603_29332_b200 as pk

    theta = mlp_init(din, H, 7)
    rng = np.random.default_rng(din + B)
    delta = (rng.normal(0, 0.3, (B, din))).astype(np.float32)
    loss, logistic, pen, gref = disc_loss_grad(theta, din, H, delta.astype(np.float64), 10.0)
    tr = pk.DiscTrainer(din, H, theta, lr=1e-3, grad_penalty=10.0, max_rows=B, math=math)
    g, lv = tr.gradient(torch.as_tensor(delta, device="cuda"))
    g, lv = g.cpu().numpy().astype(np.float64), lv.cpu().numpy()
    assert _block_rel(g, gref, din, H) <= tol_g
    assert _bias_cond_rel(g, gref, theta, din, H, delta.astype(np.float64), 10.0) <= tol_c
    assert abs(lv[0] - loss) <= tol_l * abs(loss)
    assert abs(lv[1] - logistic) <= tol_l * abs(logistic)
    assert abs(lv[2] - pen) <= max(tol_l, 3e-3 if math == 1 else 1e-4) * abs(pen)  # ||g||²: twice g's error
    tr.close()


@pytest.mark.gpu
def test_device_gradient_after_a_larger_batch():
    """Row counts change between calls (B = 999 then 37, 38, 40): the padded
    layout must not pick up rows a previous, larger batch left behind."""
    import torch

    import paper_2603_29332_b200 as pk

    din, H = 9, 16
    theta = mlp_init(din, H, 3)
    tr = pk.DiscTrainer(din, H, theta, max_rows=1000, math=0)
    tr.gradient(torch.randn(999, din, device="cuda"))
    for B in (37, 38, 40):
        d = torch.randn(B, din, device="cuda") * 0.3
        dd = d.cpu().double().numpy()
        gref = disc_loss_grad(theta, din, H, dd, 10.0)[3]
        g, _ = tr.gradient(d)
        g = g.cpu().double().numpy()
        assert _block_rel(g, gref, din, H) <= 1e-4, B
        assert _bias_cond_rel(g, gref, theta, din, H, dd, 10.0) <= 1e-5, B
    tr.close()


@pytest.mark.gpu
def test_device_gradient_ragged_rows_and_ld():
    """A Δ view with a row stride larger than its width (a rollout buffer slice), fewer rows than max_rows."""
    import torch

    import paper_2603_29332_b200 as pk

    din, H, B = 20, 32, 77
    theta = mlp_init(din, H, 5)
    full = torch.randn(B, din + 13, device="cuda") * 0.4
    view = full[:, :din]
    dd = view.cpu().double().numpy()
    gref = disc_loss_grad(theta, din, H, dd, 10.0)[3]
    tr = pk.DiscTrainer(din, H, theta, max_rows=500, math=0)
    g, _ = tr.gradient(view)
    g = g.cpu().double().numpy()
    assert _block_rel(g, gref, din, H) <= 1e-4
    assert _bias_cond_rel(g, gref, theta, din, H, dd, 10.0) <= 1e-5
    tr.close()


@pytest.mark.gpu
def test_device_adam_steps_match_oracle_and_publish():
    import torch

    import paper_2603_29332_b200 as pk
    from conftest import ensure_assets, model_paths

    ensure_assets()
    mp, cp = model_paths("wb700")
    env = pk.EnvBatch(mp, cp, 8)
    din, H, B, lr = env.delta_dim, 256, 2048, 1e-3
    theta0 = mlp_init(din, H, 7)
    rng = np.random.default_rng(9)
    batches = [(rng.normal(0, 0.2, (B, din))).astype(np.float32) for _ in range(3)]
    th_ref, adam = theta0.copy(), Adam(len(theta0), lr)
    tr = pk.DiscTrainer(din, H, theta0, lr=lr, grad_penalty=10.0, max_rows=B, math=0)
    for d in batches:
        l_ref = train_discriminator(th_ref, din, H, d.astype(np.float64), 10.0, adam)[0]
        lv = tr.step(torch.as_tensor(d, device="cuda")).cpu().numpy()
        assert abs(lv[0] - l_ref) <= 1e-5 * abs(l_ref)
    th, steps, skipped = tr.params()
    assert steps == 3 and skipped == 0
    assert np.linalg.norm(th - th_ref) <= 1e-2 * np.linalg.norm(th_ref - theta0)
    # publish into the env's reward discriminator (device repack) == set_discriminator(θ)
    env.set_discriminator(theta0, H)
    tr.publish(env)
    dx = torch.as_tensor(batches[0][:64], device="cuda")
    r = env.discriminator_reward(dx).cpu().numpy()
    ref = disc_reward(th, din, H, batches[0][:64].astype(np.float64))
    assert np.max(np.abs(r - ref) / np.maximum(1.0, np.abs(ref))) <= 3e-3
    env.set_discriminator(th, H)
    r2 = env.discriminator_reward(dx).cpu().numpy()
    assert np.array_equal(r, r2)
    tr.close()
    env.close()


@pytest.mark.gpu
def test_device_non_finite_delta_skips_the_update():
    import torch

    import paper_2603_29332_b200 as pk

    din, H = 9, 16
    theta = mlp_init(din, H, 7)
    tr = pk.DiscTrainer(din, H, theta, max_rows=16)
    d = torch.zeros(16, din, device="cuda")
    d[3, 2] = float("nan")
    tr.step(d)
    th, steps, skipped = tr.params()
    assert steps == 0 and skipped == 1 and np.array_equal(th, theta)
    tr.step(torch.zeros(16, din, device="cuda"))
    th, steps, skipped = tr.params()
    assert steps == 1 and skipped == 1 and not np.array_equal(th, theta)
    tr.close()


# ---- pins against the reference's own nn.cpp (oracle/_ref, compiled from ----
# /root/reference/proj/src/nn.cpp against the Eigen shim; golden fixture made
# from it for machines without /root/reference) --------------------------------
import os  # noqa: E402

from oracle.ref import REF_SO  # noqa: E402

HAVE_REF = os.path.exists(REF_SO)
GOLDEN_NN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "nn_reference.npz")


def _rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(1e-300, np.max(np.abs(b))))


def _nn_case(din=9, H=16, B=7, seed=11):
    rng = np.random.default_rng(seed)
    theta = mlp_init(din, H, 3)
    theta = theta + rng.normal(0, 0.05, theta.shape)  # non-zero biases
    X = rng.normal(0, 0.8, (B, din))
    up = rng.normal(0, 1.0, (B, 1))
    return theta, X, up


def _oracle_nn(theta, X, up, din, H):
    c = mlp_forward_cache(theta, din, H, X)
    from oracle.disc_train import mlp_backward

    g_b = np.zeros(theta.size)
    ig = mlp_backward(c, up, g_b, din, H, input_grad=True)
    g_p = np.zeros(theta.size)
    pen = gradient_penalty_backward(c, g_p, din, H)
    return c["y"], g_b, ig, g_p, pen


@pytest.mark.skipif(not HAVE_REF, reason="reference build oracle/_ref absent")
@pytest.mark.parametrize("din,H,B", [(9, 16, 7), (102, 64, 33)])
def test_oracle_mlp_matches_reference_nn_cpp(din, H, B):
    """Mlp::forward / Mlp::backward / Mlp::gradient_penalty_backward of the
    REFERENCE (nn.cpp:54-222) equal the oracle restatement (oracle/disc_train.py)
    to f64 rounding (different summation order only)."""
    from oracle.ref import ref_mlp_backward, ref_mlp_forward, ref_mlp_gp_backward, ref_mlp_init

    assert np.array_equal(ref_mlp_init(din, H, 1, 3), mlp_init(din, H, 3))  # Mlp(shape, seed)
    theta, X, up = _nn_case(din, H, B)
    y, g_b, ig, g_p, pen = _oracle_nn(theta, X, up, din, H)
    assert _rel(y, ref_mlp_forward(theta, din, H, 1, X)) <= 1e-14
    rg, rig = ref_mlp_backward(theta, din, H, 1, X, up)
    assert _rel(g_b, rg) <= 1e-12 and _rel(ig, rig) <= 1e-12
    rgp, rpen = ref_mlp_gp_backward(theta, din, H, X)
    assert _rel(g_p, rgp) <= 1e-12 and _rel(pen, rpen) <= 1e-12


@pytest.mark.skipif(not HAVE_REF, reason="reference build oracle/_ref absent")
def test_oracle_adam_and_running_norm_match_reference():
    """Adam::step (nn.cpp:224-240, incl. the non-finite skip) and RunningNorm
    update/apply (nn.cpp:246-277) of the reference vs the oracles."""
    from oracle.ref import RefAdam, ref_running_norm

    import paper_2603_29332_b200.dist as pkd
    from oracle.policy import running_norm_apply

    rng = np.random.default_rng(2)
    n = 50
    p_o, p_r = rng.normal(0, 1, n), None
    p_r = p_o.copy()
    a_o, a_r = Adam(n, 3e-3), RefAdam(n, 3e-3)
    for k in range(4):
        g = rng.normal(0, 1, n)
        if k == 2:
            g[5] = np.nan  # skipped by both
        assert a_o.step(p_o, g) == a_r.step(p_r, g)
    assert _rel(p_o, p_r) <= 1e-15 and a_o.skipped == a_r.skipped.value == 1
    cnt, mean, var = 0.0, np.zeros(6), np.ones(6)
    for k in range(3):
        X = rng.normal(k, 1.0 + k, (20 + k, 6))
        rc, rm, rv, ry = ref_running_norm(X, cnt, mean, var)
        m = pkd.batch_moments(__import__("torch").as_tensor(X)).numpy()
        cnt, mean, var = pkd.running_norm_fold(cnt, mean, var, m[0], m[1:7], m[7:])
        assert cnt == rc and _rel(mean, rm) <= 1e-14 and _rel(var, rv) <= 1e-13
        assert _rel(running_norm_apply(X, mean, var, cnt), ry) <= 1e-13


def test_oracle_mlp_reproduces_reference_golden():
    """The same pins from the committed fixture (made by the reference build,
    tests/golden/make_golden.py) where /root/reference is absent."""
    g = np.load(GOLDEN_NN)
    din, H = int(g["shape"][0]), int(g["shape"][1])
    y, g_b, ig, g_p, pen = _oracle_nn(g["theta"], g["X"], g["up"], din, H)
    assert _rel(y, g["y"]) <= 1e-14
    assert _rel(g_b, g["grad_backward"]) <= 1e-12 and _rel(ig, g["input_grad"]) <= 1e-12
    assert _rel(g_p, g["grad_penalty"]) <= 1e-12 and _rel(pen, g["penalty"]) <= 1e-12


def test_oracle_bias_adjoint_rows_sum_to_the_gradient():
    """bias_adjoint_rows (the conditioning measure of the bias-block checks) sums to
    disc_loss_grad's bias gradients, and the D(0) row cancels most of the Δ rows."""
    from oracle.disc_train import bias_adjoint_rows

    din, H, B = 9, 16, 37
    theta = mlp_init(din, H, 7)
    delta = np.random.default_rng(1).normal(0, 0.3, (B, din))
    g = disc_loss_grad(theta, din, H, delta, 10.0)[3]
    rows = bias_adjoint_rows(theta, din, H, delta, 10.0)
    for (a, b), rw in zip(_blocks(din, H)[1::2], rows):
        assert rw.shape == (B + 1, b - a)
        assert np.max(np.abs(rw.sum(0) - g[a:b])) <= 1e-15
        assert np.linalg.norm(np.abs(rw).sum(0)) > 50 * np.linalg.norm(g[a:b])


@pytest.mark.gpu
@pytest.mark.parametrize("din,H,B", [(9, 16, 37), (102, 256, 300)])
def test_trainer_outputs_stay_inside_caller_buffers(din, H, B):
    """Out-of-bounds check for the training step's caller buffers (compute-sanitizer
    is closed on the GPU pool): grad / loss outputs and the Δ input view sit inside
    larger buffers whose guard bytes must survive gradient() and step()."""
    import ctypes as C

    import torch

    import paper_2603_29332_b200 as pk

    GUARD = 4096
    theta = mlp_init(din, H, 7)
    tr = pk.DiscTrainer(din, H, theta, max_rows=B, math=0)
    P = len(theta)
    graw = torch.full((P + 2 * GUARD,), -7.0, device="cuda")
    lraw = torch.full((3 + 2 * GUARD,), -7.0, dtype=torch.float64, device="cuda")
    draw = torch.full(((B + 2) * (din + 3),), -7.0, device="cuda")
    delta = draw[(din + 3):(B + 1) * (din + 3)].view(B, din + 3)[:, :din]  # strided view, guards around
    delta.copy_(torch.randn(B, din, device="cuda") * 0.3)
    L = pk.lib()
    for _ in range(2):
        assert L.msk_disc_trainer_gradient(tr.h_, C.c_void_p(delta.data_ptr()), B, delta.stride(0),
                                           C.c_void_p(graw.data_ptr() + 4 * GUARD),
                                           C.c_void_p(lraw.data_ptr() + 8 * GUARD),
                                           C.c_void_p(torch.cuda.current_stream().cuda_stream)) == 0
        tr.step(delta)
    torch.cuda.synchronize()
    for raw, n in ((graw, P), (lraw, 3)):
        assert torch.all(raw[:GUARD] == -7.0) and torch.all(raw[GUARD + n:] == -7.0)
    assert torch.all(draw[:din + 3] == -7.0) and torch.all(draw[(B + 1) * (din + 3):] == -7.0)
    assert torch.all(torch.isfinite(graw[GUARD:GUARD + P]))
    tr.close()
