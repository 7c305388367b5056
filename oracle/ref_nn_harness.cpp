// TEST INFRASTRUCTURE ONLY — drives the reference's own nn.cpp (compiled from
// /root/reference/proj/src against oracle/shim, see oracle/Makefile) through a
// C ABI, so the discriminator / policy restatements (oracle/disc_train.py,
// oracle/policy.py, oracle/msk_oracle.c) are pinned to Mlp::forward,
// Mlp::backward, Mlp::gradient_penalty_backward and Adam::step themselves
// (nn.cpp:16-244).  Matrices cross the ABI row-major (batch x features).
#include <cstdint>
#include <cstring>

#include "msk/nn.hpp"

namespace {

msk::Mlp make_mlp(const double* theta, int64_t n, int in, int hidden, int out, int head, double aff_s,
                  double aff_o) {
    msk::MlpShape sh;
    sh.in = in;
    sh.hidden = hidden;
    sh.out = out;
    sh.head = static_cast<msk::Head>(head);
    sh.affine_scale = aff_s;
    sh.affine_offset = aff_o;
    msk::Mlp m(sh, 0);
    if (theta) {
        if (m.param_count() != n) return m;
        for (int64_t i = 0; i < n; ++i) m.params()[i] = theta[i];
    }
    return m;
}

Eigen::MatrixXd from_rows(const double* x, int rows, int cols) {
    Eigen::MatrixXd m = Eigen::MatrixXd::Zero(rows, cols);
    for (int i = 0; i < rows; ++i)
        for (int j = 0; j < cols; ++j) m(i, j) = x[static_cast<size_t>(i) * cols + j];
    return m;
}

void to_rows(const Eigen::MatrixXd& m, double* out) {
    for (Eigen::Index i = 0; i < m.rows(); ++i)
        for (Eigen::Index j = 0; j < m.cols(); ++j) out[static_cast<size_t>(i) * m.cols() + j] = m(i, j);
}

}  // namespace

extern "C" {

// Mlp(MlpShape{in, hidden, out, head, ..., final_init_scale}, seed) parameters (nn.cpp:16-38).
int64_t ref_mlp_init(int32_t in, int32_t hidden, int32_t out, uint64_t seed, double final_init_scale, double* theta) {
    msk::MlpShape sh;
    sh.in = in;
    sh.hidden = hidden;
    sh.out = out;
    sh.final_init_scale = final_init_scale;
    msk::Mlp m(sh, seed);
    if (theta) std::memcpy(theta, m.params().data(), sizeof(double) * m.param_count());
    return m.param_count();
}

// Mlp::forward (nn.cpp:54-73): Y [B x out].
void ref_mlp_forward(const double* theta, int64_t n, int32_t in, int32_t hidden, int32_t out, int32_t head,
                     double aff_s, double aff_o, const double* X, int32_t B, double* Y) {
    const msk::Mlp m = make_mlp(theta, n, in, hidden, out, head, aff_s, aff_o);
    to_rows(m.forward(from_rows(X, B, in)), Y);
}

// Mlp::backward (nn.cpp:80-129): grad [n] accumulated (caller zeroes it),
// input_grad [B x in] (nullable).
void ref_mlp_backward(const double* theta, int64_t n, int32_t in, int32_t hidden, int32_t out, int32_t head,
                      double aff_s, double aff_o, const double* X, int32_t B, const double* upstream, double* grad,
                      double* input_grad) {
    const msk::Mlp m = make_mlp(theta, n, in, hidden, out, head, aff_s, aff_o);
    msk::Mlp::Cache c;
    m.forward(from_rows(X, B, in), c);
    Eigen::VectorXd g = Eigen::VectorXd::Zero(n);
    for (int64_t i = 0; i < n; ++i) g[i] = grad[i];
    Eigen::MatrixXd ig;
    m.backward(c, from_rows(upstream, B, out), g, input_grad ? &ig : nullptr);
    for (int64_t i = 0; i < n; ++i) grad[i] = g[i];
    if (input_grad) to_rows(ig, input_grad);
}

// Mlp::gradient_penalty_backward (nn.cpp:131-222): grad [n] accumulated,
// penalty [B] = ||dy/dx||^2 per sample.
void ref_mlp_gp_backward(const double* theta, int64_t n, int32_t in, int32_t hidden, int32_t head,
                         const double* X, int32_t B, double* grad, double* penalty) {
    const msk::Mlp m = make_mlp(theta, n, in, hidden, 1, head, 1.0, 0.0);
    msk::Mlp::Cache c;
    m.forward(from_rows(X, B, in), c);
    Eigen::VectorXd g = Eigen::VectorXd::Zero(n);
    for (int64_t i = 0; i < n; ++i) g[i] = grad[i];
    const Eigen::VectorXd p = m.gradient_penalty_backward(c, g);
    for (int64_t i = 0; i < n; ++i) grad[i] = g[i];
    for (int32_t i = 0; i < B; ++i) penalty[i] = p[i];
}

// Adam::step (nn.cpp:224-240) on caller-held state; returns 1 if applied, 0 if skipped.
int32_t ref_adam_step(double* params, const double* grad, int64_t n, double lr, double* m, double* v,
                      int64_t* step_count, int64_t* skipped) {
    msk::Adam a(static_cast<int>(n), lr);
    a.step_count = static_cast<long>(*step_count);
    a.skipped = static_cast<long>(*skipped);
    Eigen::VectorXd p = Eigen::VectorXd::Zero(n), g = Eigen::VectorXd::Zero(n);
    for (int64_t i = 0; i < n; ++i) {
        p[i] = params[i];
        g[i] = grad[i];
        a.m[i] = m[i];
        a.v[i] = v[i];
    }
    const bool ok = a.step(p, g);
    for (int64_t i = 0; i < n; ++i) {
        params[i] = p[i];
        m[i] = a.m[i];
        v[i] = a.v[i];
    }
    *step_count = a.step_count;
    *skipped = a.skipped;
    return ok ? 1 : 0;
}

// RunningNorm::update then apply (nn.cpp:246-284): X [B x D]; state (count,
// mean, var) in/out; Y [B x D] = apply(X) after the update.
void ref_running_norm(const double* X, int32_t B, int32_t D, double* count, double* mean, double* var, double* Y) {
    msk::RunningNorm rn(D);
    rn.count = *count;
    for (int32_t j = 0; j < D; ++j) {
        rn.mean[j] = mean[j];
        rn.var[j] = var[j];
    }
    const Eigen::MatrixXd x = from_rows(X, B, D);
    rn.update(x);
    to_rows(rn.apply(x), Y);
    *count = rn.count;
    for (int32_t j = 0; j < D; ++j) {
        mean[j] = rn.mean[j];
        var[j] = rn.var[j];
    }
}

}  // extern "C"
