"""Oracle (test infrastructure only): f64 restatement of the discriminator
training step — SPEC.md:412-421 train_discriminator on the nn.cpp Mlp.

  loss = -log clamp(D(0)) - mean_i log(1 - clamp(D(Δ_i))) + λ mean_i ||∇_Δ D(Δ_i)||²

D = Mlp(in = dΔ, hidden = W, out = 1, Head::Sigmoid), clamp to [1e-4, 1 - 1e-4]
inside the logs, gradient penalty at the sampled Δ points
(one-sided), then one Adam step (nn.cpp:224-240; β1 0.9, β2 0.999,
ε 1e-8, nn.hpp:78; a non-finite gradient skips the step).

Functions follow the reference line by line:
  mlp_forward_cache        nn.cpp:54-73   (Mlp::forward with Cache)
  mlp_backward             nn.cpp:80-129  (Mlp::backward, sigmoid head)
  gradient_penalty_backward nn.cpp:131-222 (forward tangent along g = dy/dx, reverse pass)
  adam_step                nn.cpp:224-240
The clamp's derivative is taken as 0 outside [1e-4, 1 - 1e-4] (its subgradient);
learn.cpp, which would compose these calls, is absent from the reference.

Parity status: pinned to the reference itself — nn.cpp is compiled unchanged
into oracle/_ref (the Eigen shim provides its Map / Array / rowwise / colwise
API) and Mlp::forward / backward / gradient_penalty_backward, Adam::step and
RunningNorm agree with these functions to <= 1e-12 relative
(tests/test_disc_train.py, and tests/golden/nn_reference.npz where
/root/reference is absent); finite-difference gradient checks
and SPEC.md:419-420's examples are kept.  The composition into the loss
(train_discriminator) follows SPEC.md:412-421, learn.cpp being absent.
"""
import numpy as np

from .policy import mlp_layers

CLAMP_LO, CLAMP_HI = 1e-4, 1.0 - 1e-4


def _flat_offsets(n_in, hidden, n_out=1):
    dims = [(hidden, n_in), (hidden, hidden), (hidden, hidden), (n_out, hidden)]
    offs, o = [], 0
    for r, c in dims:
        offs.append((o, o + r * c, r, c))
        o += r * c + r
    return offs, o


def mlp_forward_cache(theta, n_in, hidden, X):
    """Mlp::forward(X, cache) with Head::Sigmoid (nn.cpp:54-73): returns cache dict."""
    L = mlp_layers(theta, n_in, hidden, 1)
    X = np.asarray(X, dtype=np.float64)
    h1 = np.tanh(X @ L[0][0].T + L[0][1])
    h2 = np.tanh(h1 @ L[1][0].T + L[1][1])
    h3 = np.tanh(h2 @ L[2][0].T + L[2][1])
    z = h3 @ L[3][0].T + L[3][1]
    y = 1.0 / (1.0 + np.exp(-z))
    return {"x": X, "h1": h1, "h2": h2, "h3": h3, "y": y, "layers": L}


def _grad_views(grad, n_in, hidden):
    offs, _ = _flat_offsets(n_in, hidden)
    views = []
    for w0, b0, r, c in offs:
        Wv = grad[w0:w0 + r * c].reshape(c, r).T  # column-major view (writes land in grad)
        bv = grad[b0:b0 + r]
        views.append((Wv, bv))
    return views


def mlp_backward(cache, upstream, grad, n_in, hidden, input_grad=False):
    """Mlp::backward (nn.cpp:80-129), sigmoid head: accumulates into grad (flat, f64)."""
    L, y = cache["layers"], cache["y"]
    g = _grad_views(grad, n_in, hidden)
    dz4 = upstream * y * (1.0 - y)
    g[3][0][...] += dz4.T @ cache["h3"]
    g[3][1][...] += dz4.sum(axis=0)
    dz3 = (dz4 @ L[3][0]) * (1.0 - cache["h3"] ** 2)
    g[2][0][...] += dz3.T @ cache["h2"]
    g[2][1][...] += dz3.sum(axis=0)
    dz2 = (dz3 @ L[2][0]) * (1.0 - cache["h2"] ** 2)
    g[1][0][...] += dz2.T @ cache["h1"]
    g[1][1][...] += dz2.sum(axis=0)
    dz1 = (dz2 @ L[1][0]) * (1.0 - cache["h1"] ** 2)
    g[0][0][...] += dz1.T @ cache["x"]
    g[0][1][...] += dz1.sum(axis=0)
    return dz1 @ L[0][0] if input_grad else None


def gradient_penalty_backward(cache, grad, n_in, hidden):
    """Mlp::gradient_penalty_backward (nn.cpp:131-222): accumulates d(Σ_i ||g_i||²)/dθ
    into grad and returns penalty_i = ||dy_i/dx_i||²."""
    L, y = cache["layers"], cache["y"][:, 0]
    W = [l[0] for l in L]
    d4 = y * (1.0 - y)
    dd4 = d4 * (1.0 - 2.0 * y)
    h1, h2, h3, x = cache["h1"], cache["h2"], cache["h3"], cache["x"]
    g1, g2, g3 = 1.0 - h1 ** 2, 1.0 - h2 ** 2, 1.0 - h3 ** 2
    d3 = (d4[:, None] * W[3]) * g3
    d2 = (d3 @ W[2]) * g2
    d1 = (d2 @ W[1]) * g1
    gx = d1 @ W[0]
    zeta1 = gx @ W[0].T
    u1 = g1 * zeta1
    zeta2 = u1 @ W[1].T
    u2 = g2 * zeta2
    zeta3 = u2 @ W[2].T
    u3 = g3 * zeta3
    zeta4 = (u3 @ W[3].T)[:, 0]
    penalty = d4 * zeta4
    gv = _grad_views(grad, n_in, hidden)
    b_zeta4 = 2.0 * d4
    b_z4 = 2.0 * dd4 * zeta4
    gv[3][0][...] += b_zeta4[None, :] @ u3 + b_z4[None, :] @ h3
    gv[3][1][...] += b_z4.sum()
    b_u3 = b_zeta4[:, None] * W[3]
    b_h3 = b_z4[:, None] * W[3]
    b_zeta3 = g3 * b_u3
    b_h3 = b_h3 - 2.0 * h3 * zeta3 * b_u3
    b_z3 = g3 * b_h3
    gv[2][0][...] += b_zeta3.T @ u2 + b_z3.T @ h2
    gv[2][1][...] += b_z3.sum(axis=0)
    b_u2, b_h2 = b_zeta3 @ W[2], b_z3 @ W[2]
    b_zeta2 = g2 * b_u2
    b_h2 = b_h2 - 2.0 * h2 * zeta2 * b_u2
    b_z2 = g2 * b_h2
    gv[1][0][...] += b_zeta2.T @ u1 + b_z2.T @ h1
    gv[1][1][...] += b_z2.sum(axis=0)
    b_u1, b_h1 = b_zeta2 @ W[1], b_z2 @ W[1]
    b_zeta1 = g1 * b_u1
    b_h1 = b_h1 - 2.0 * h1 * zeta1 * b_u1
    b_z1 = g1 * b_h1
    gv[0][0][...] += b_zeta1.T @ gx + b_z1.T @ x
    gv[0][1][...] += b_z1.sum(axis=0)
    return penalty


class Adam:
    """Adam (nn.cpp:224-240, nn.hpp:76-82)."""

    def __init__(self, n, lr, beta1=0.9, beta2=0.999, eps=1e-8):
        self.lr, self.beta1, self.beta2, self.eps = lr, beta1, beta2, eps
        self.m, self.v = np.zeros(n), np.zeros(n)
        self.step_count, self.skipped = 0, 0

    def step(self, params, grad):
        if not np.all(np.isfinite(grad)):
            self.skipped += 1
            return False
        self.step_count += 1
        self.m = self.beta1 * self.m + (1.0 - self.beta1) * grad
        self.v = self.beta2 * self.v + (1.0 - self.beta2) * grad * grad
        bc1 = 1.0 - self.beta1 ** self.step_count
        bc2 = 1.0 - self.beta2 ** self.step_count
        params -= self.lr * (self.m / bc1) / (np.sqrt(self.v / bc2) + self.eps)
        return True


def disc_loss_grad(theta, n_in, hidden, delta, lam):
    """Loss terms and dloss/dθ of train_discriminator at theta.
    Returns (loss, logistic, penalty_mean, grad)."""
    delta = np.asarray(delta, dtype=np.float64)
    B = delta.shape[0]
    grad = np.zeros(len(theta))
    # -log clamp(D(0))
    c0 = mlp_forward_cache(theta, n_in, hidden, np.zeros((1, n_in)))
    y0 = c0["y"][0, 0]
    inside0 = CLAMP_LO < y0 < CLAMP_HI
    mlp_backward(c0, np.array([[-1.0 / y0 if inside0 else 0.0]]), grad, n_in, hidden)
    # -mean log(1 - clamp(D(Δ)))
    c = mlp_forward_cache(theta, n_in, hidden, delta)
    y = c["y"][:, 0]
    yc = np.clip(y, CLAMP_LO, CLAMP_HI)
    inside = (y > CLAMP_LO) & (y < CLAMP_HI)
    up = np.where(inside, 1.0 / (1.0 - y), 0.0) / B
    mlp_backward(c, up[:, None], grad, n_in, hidden)
    logistic = -np.log(np.clip(y0, CLAMP_LO, CLAMP_HI)) - np.mean(np.log(1.0 - yc))
    pen_mean = 0.0
    if lam != 0.0:
        gp = np.zeros(len(theta))
        pen = gradient_penalty_backward(c, gp, n_in, hidden)
        grad += (lam / B) * gp
        pen_mean = float(np.mean(pen))
    return logistic + lam * pen_mean, logistic, pen_mean, grad


def bias_adjoint_rows(theta, n_in, hidden, delta, lam):
    """Per-row bias adjoints of dloss/dθ (the rows whose column sums are the
    bias gradients of disc_loss_grad): [b0 rows, b1 rows, b2 rows, b4 rows], each
    [(B + 1) x out], Δ rows first, then the D(0) row.  Used to state the
    conditioning of the bias gradients (Σ_r |row| vs |Σ_r row|: the D(0) term
    cancels most of the Δ terms), nn.cpp:98-128 and 186-221 row by row."""
    delta = np.asarray(delta, dtype=np.float64)
    B = delta.shape[0]
    L = mlp_layers(theta, n_in, hidden, 1)
    W = [l[0] for l in L]

    def logistic_rows(c, upstream):
        y = c["y"]
        dz4 = upstream * y * (1.0 - y)
        dz3 = (dz4 @ W[3]) * (1.0 - c["h3"] ** 2)
        dz2 = (dz3 @ W[2]) * (1.0 - c["h2"] ** 2)
        dz1 = (dz2 @ W[1]) * (1.0 - c["h1"] ** 2)
        return [dz1, dz2, dz3, dz4]

    c0 = mlp_forward_cache(theta, n_in, hidden, np.zeros((1, n_in)))
    y0 = c0["y"][0, 0]
    z0 = logistic_rows(c0, np.array([[-1.0 / y0 if CLAMP_LO < y0 < CLAMP_HI else 0.0]]))
    c = mlp_forward_cache(theta, n_in, hidden, delta)
    y = c["y"][:, 0]
    inside = (y > CLAMP_LO) & (y < CLAMP_HI)
    zr = logistic_rows(c, (np.where(inside, 1.0 / (1.0 - y), 0.0) / B)[:, None])
    if lam != 0.0:
        d4 = y * (1.0 - y)
        dd4 = d4 * (1.0 - 2.0 * y)
        h1, h2, h3 = c["h1"], c["h2"], c["h3"]
        g1, g2, g3 = 1.0 - h1 ** 2, 1.0 - h2 ** 2, 1.0 - h3 ** 2
        d3 = (d4[:, None] * W[3]) * g3
        d1 = (((d3 @ W[2]) * g2) @ W[1]) * g1
        zeta1 = (d1 @ W[0]) @ W[0].T
        u1 = g1 * zeta1
        zeta2 = u1 @ W[1].T
        u2 = g2 * zeta2
        zeta3 = u2 @ W[2].T
        zeta4 = ((g3 * zeta3) @ W[3].T)[:, 0]
        w = lam / B
        b_u3, b_h3 = (w * 2.0 * d4)[:, None] * W[3], (w * 2.0 * dd4 * zeta4)[:, None] * W[3]
        b_z4 = (w * 2.0 * dd4 * zeta4)[:, None]
        b_zeta3, b_z3 = g3 * b_u3, g3 * (b_h3 - 2.0 * h3 * zeta3 * b_u3)
        b_u2, b_h2 = b_zeta3 @ W[2], b_z3 @ W[2]
        b_zeta2, b_z2 = g2 * b_u2, g2 * (b_h2 - 2.0 * h2 * zeta2 * b_u2)
        b_u1, b_h1 = b_zeta2 @ W[1], b_z2 @ W[1]
        b_z1 = g1 * (b_h1 - 2.0 * h1 * zeta1 * b_u1)
        for k, pz in enumerate([b_z1, b_z2, b_z3, b_z4]):
            zr[k] = zr[k] + pz
    return [np.vstack([a, b]) for a, b in zip(zr, z0)]


def train_discriminator(theta, n_in, hidden, delta, lam, adam):
    """One update: returns (loss, logistic, penalty) at the
    pre-update parameters; theta is updated in place by adam."""
    loss, logistic, pen, grad = disc_loss_grad(theta, n_in, hidden, delta, lam)
    adam.step(theta, grad)
    return loss, logistic, pen
