"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the parity checkers.

* ``RefBatch``    drives the reference's own msk::Env, compiled unchanged from
                  /root/reference/proj/src (oracle/_ref/libmsk_ref.so, built by
                  oracle/Makefile against oracle/shim/Eigen).
* ``OracleBatch`` drives the plain-C restatement (oracle/libmsk_oracle.so).

Both expose the same batched verbs (reset / reset_to_frame / step / state
get+set / sampler / outcomes) with float64 numpy buffers so the tests can
compare them with each other and with the CUDA path.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu-baseline leg may import this.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libmsk_ref.so")
# the same sources built for speed (-O3, FMA contraction): the CPU timing arm only
REF_FAST_SO = os.path.join(HERE, "_ref", "libmsk_ref_fast.so")
ORACLE_SO = os.path.join(HERE, "libmsk_oracle.so")

FLAG_DONE, FLAG_FAILED, FLAG_DIVERGED, FLAG_NOT_STEPPED, FLAG_BAD_ACTION = 1, 2, 4, 8, 16

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_up = C.POINTER(C.c_uint8)


class EnvConfigC(C.Structure):
    _fields_ = [
        ("episode_horizon", C.c_int32),
        ("rsi", C.c_int32),
        ("adaptive_bins", C.c_int32),
        ("pad0", C.c_int32),
        ("adaptive_mix", C.c_double),
        ("adaptive_decay", C.c_double),
        ("termination_body_err", C.c_double),
        ("init_activation", C.c_double),
    ]


class RewardConfigC(C.Structure):
    _fields_ = [
        ("mode", C.c_int32),
        ("n_emg_channels", C.c_int32),
        ("w_emg", C.c_double),
        ("w_power", C.c_double),
        ("emg_channel_map", _ip),
    ]


def env_config(episode_horizon=250, rsi=True, adaptive_bins=10, adaptive_mix=0.2, adaptive_decay=0.99,
               termination_body_err=0.5, init_activation=0.01):
    """Defaults of msk::EnvConfig (/root/reference/proj/include/msk/env.hpp:39-47)."""
    return EnvConfigC(int(episode_horizon), int(bool(rsi)), int(adaptive_bins), 0, float(adaptive_mix),
                      float(adaptive_decay), float(termination_body_err), float(init_activation))


def _ptr(a, t):
    return a.ctypes.data_as(t) if a is not None else None


def _load(path):
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing — run `make -C oracle` (or __graft_entry__.build())")
    return C.CDLL(path)


_REF = {}


def ref_lib(fast=False):
    """The reference build (fast=True: the -O3 / FMA-contracted build used to time
    the CPU arm; parity checks always use the strict-IEEE build)."""
    path = REF_FAST_SO if fast else REF_SO
    if path not in _REF:
        lib = _load(path)
        lib.ref_create.restype = C.c_void_p
        lib.ref_create.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(EnvConfigC), C.POINTER(RewardConfigC),
                                   C.c_int32, C.c_uint64, C.c_int64, C.c_char_p, C.c_int32]
        lib.ref_destroy.argtypes = [C.c_void_p]
        lib.ref_dims.argtypes = [C.c_void_p, _ip]
        lib.ref_set_threads.argtypes = [C.c_void_p, C.c_int32]
        lib.ref_set_eval_mode.argtypes = [C.c_void_p, C.c_int32]
        lib.ref_reset.argtypes = [C.c_void_p, _up, _dp, _ip, C.c_char_p, C.c_int32]
        lib.ref_reset_to_frame.argtypes = [C.c_void_p, _ip, _up, _dp, C.c_char_p, C.c_int32]
        lib.ref_step.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _up, _dp, _dp]
        lib.ref_observe.argtypes = [C.c_void_p, _dp]
        lib.ref_tracking_error.argtypes = [C.c_void_p, _dp]
        lib.ref_force_state_to_reference.argtypes = [C.c_void_p]
        lib.ref_get_state.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _ip]
        lib.ref_set_state.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _ip]
        lib.ref_get_sampler.argtypes = [C.c_void_p, _dp]
        lib.ref_set_sampler.argtypes = [C.c_void_p, _dp]
        lib.ref_record_own_outcomes.argtypes = [C.c_void_p]
        lib.ref_drain_outcomes.argtypes = [C.c_void_p, _ip, _up, _ip, C.c_int32]
        lib.ref_rng_raw.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_uint64)]
        P = C.POINTER
        lib.ref_mlp_init.restype = C.c_int64
        lib.ref_mlp_init.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_uint64, C.c_double, _dp]
        lib.ref_mlp_forward.argtypes = [_dp, C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_double,
                                        C.c_double, _dp, C.c_int32, _dp]
        lib.ref_mlp_backward.argtypes = [_dp, C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_double,
                                         C.c_double, _dp, C.c_int32, _dp, _dp, _dp]
        lib.ref_mlp_gp_backward.argtypes = [_dp, C.c_int64, C.c_int32, C.c_int32, C.c_int32, _dp, C.c_int32, _dp,
                                            _dp]
        lib.ref_adam_step.restype = C.c_int32
        lib.ref_adam_step.argtypes = [_dp, _dp, C.c_int64, C.c_double, _dp, _dp, P(C.c_int64), P(C.c_int64)]
        lib.ref_running_norm.argtypes = [_dp, C.c_int32, C.c_int32, _dp, _dp, _dp, _dp]
        lib.ref_rng_serialize.restype = C.c_int32
        lib.ref_rng_serialize.argtypes = [C.c_void_p, C.c_int32, C.c_char_p, C.c_int32]
        lib.ref_rng_deserialize.argtypes = [C.c_void_p, C.c_int32, C.c_char_p]
        lib.ref_excitations.argtypes = [C.c_uint64, C.c_uint32, C.c_int64, C.c_int32, C.c_int32, _dp]
        lib.ref_rng_uniform.argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_int64, _dp]
        lib.ref_bench.restype = C.c_double
        lib.ref_bench.argtypes = [C.c_void_p, C.c_int32, C.c_uint64, C.POINTER(C.c_int64)]
        lib.ref_set_discriminator.argtypes = [C.c_void_p, _dp, C.c_int64, C.c_int32]
        lib.ref_set_discriminator.restype = C.c_int32
        for fn in ("ref_force_length_active", "ref_force_velocity", "ref_force_passive", "ref_wrap_angle"):
            getattr(lib, fn).restype = C.c_double
            getattr(lib, fn).argtypes = [C.c_double]
        lib.ref_mtu_force.restype = C.c_double
        lib.ref_mtu_force.argtypes = [C.c_double] * 4
        lib.ref_activation_step.restype = C.c_double
        lib.ref_activation_step.argtypes = [C.c_double] * 5
        lib.ref_mass_matrix.argtypes = [C.c_void_p, _dp, _dp]
        lib.ref_moment_arms.argtypes = [C.c_void_p, _dp, _dp]
        lib.ref_bias_forces.argtypes = [C.c_void_p, _dp, _dp, _dp]
        lib.ref_mtu_length.restype = C.c_double
        lib.ref_mtu_length.argtypes = [C.c_void_p, _dp, C.c_int32]
        lib.ref_mechanical_energy.restype = C.c_double
        lib.ref_mechanical_energy.argtypes = [C.c_void_p, _dp, _dp]
        lib.ref_key_bodies.argtypes = [C.c_void_p, _dp, _dp, _dp]
        _REF[path] = lib
    return _REF[path]


def excitations(seed, step, n_envs, nm, global_env_offset=0):
    """Philox4x32-10 excitations, as float64 (E x nm)."""
    out = np.zeros((n_envs, nm), dtype=np.float64)
    ref_lib().ref_excitations(C.c_uint64(seed), C.c_uint32(step), C.c_int64(global_env_offset), n_envs, nm,
                              _ptr(out, _dp))
    return out


class RefBatch:
    """E independent reference ``msk::Env`` instances (seed = base_seed + global index)."""

    def __init__(self, model_path, clip_path, n_envs, base_seed=0x5EED, cfg=None, reward_mode=0, w_emg=100.0,
                 w_power=0.05, emg_map=(), global_env_offset=0, threads=1, fast=False):
        lib = ref_lib(fast)
        self.lib = lib
        cfg = cfg if cfg is not None else env_config()
        self._emg = np.asarray(emg_map, dtype=np.int32)
        rc = RewardConfigC(int(reward_mode), len(self._emg), float(w_emg), float(w_power),
                           _ptr(self._emg, _ip) if len(self._emg) else None)
        err = C.create_string_buffer(512)
        self.h = lib.ref_create(model_path.encode(), (clip_path or "").encode(), C.byref(cfg), C.byref(rc),
                                n_envs, C.c_uint64(base_seed), global_env_offset, err, 512)
        if not self.h:
            raise RuntimeError(err.value.decode())
        dims = np.zeros(10, dtype=np.int32)
        lib.ref_dims(self.h, _ptr(dims, _ip))
        (self.nq, self.nm, self.obs_dim, self.delta_dim, self.n_links, self.frames, self.nk, self.nj,
         floating, self.n_spheres) = [int(x) for x in dims]
        self.floating = bool(floating)
        self.n = n_envs
        self.bins = int(cfg.adaptive_bins)
        if threads > 1:
            lib.ref_set_threads(self.h, threads)

    def close(self):
        if self.h:
            self.lib.ref_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_eval_mode(self, ev=True):
        self.lib.ref_set_eval_mode(self.h, int(bool(ev)))

    def reset(self, mask=None):
        obs = np.zeros((self.n, self.obs_dim))
        frames = np.full(self.n, -1, dtype=np.int32)
        m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
        err = C.create_string_buffer(512)
        if self.lib.ref_reset(self.h, _ptr(m, _up), _ptr(obs, _dp), _ptr(frames, _ip), err, 512):
            raise RuntimeError(err.value.decode())
        return obs, frames

    def reset_to_frame(self, frames, mask=None):
        fr = np.ascontiguousarray(np.broadcast_to(np.asarray(frames, dtype=np.int32), (self.n,)))
        obs = np.zeros((self.n, self.obs_dim))
        m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
        err = C.create_string_buffer(512)
        if self.lib.ref_reset_to_frame(self.h, _ptr(fr, _ip), _ptr(m, _up), _ptr(obs, _dp), err, 512):
            raise RuntimeError(err.value.decode())
        return obs

    def step(self, actions):
        a = np.ascontiguousarray(actions, dtype=np.float64).reshape(self.n, self.nm)
        obs = np.zeros((self.n, self.obs_dim))
        delta = np.zeros((self.n, self.delta_dim))
        raux = np.zeros(self.n)
        flags = np.zeros(self.n, dtype=np.uint8)
        power = np.zeros((self.n, self.nm))
        grf = np.zeros((self.n, self.n_links, 2))
        self.lib.ref_step(self.h, _ptr(a, _dp), _ptr(obs, _dp), _ptr(delta, _dp), _ptr(raux, _dp),
                          _ptr(flags, _up), _ptr(power, _dp), _ptr(grf, _dp))
        return dict(obs=obs, delta=delta, reward_aux=raux, flags=flags, power=power, grf=grf)

    def observe(self):
        obs = np.zeros((self.n, self.obs_dim))
        self.lib.ref_observe(self.h, _ptr(obs, _dp))
        return obs

    def tracking_error(self):
        d = np.zeros((self.n, self.delta_dim))
        self.lib.ref_tracking_error(self.h, _ptr(d, _dp))
        return d

    def force_state_to_reference(self):
        self.lib.ref_force_state_to_reference(self.h)

    def get_state(self):
        n, nq, nm = self.n, self.nq, self.nm
        s = dict(q=np.zeros((n, nq)), dq=np.zeros((n, nq)), act=np.zeros((n, nm)), l_m=np.zeros((n, nm)),
                 v_m=np.zeros((n, nm)), f_m=np.zeros((n, nm)), t=np.zeros(n), ints=np.zeros((n, 4), dtype=np.int32))
        self.lib.ref_get_state(self.h, *[_ptr(s[k], _dp) for k in ("q", "dq", "act", "l_m", "v_m", "f_m", "t")],
                               _ptr(s["ints"], _ip))
        return s

    def set_state(self, s):
        arrs = [np.ascontiguousarray(s[k], dtype=np.float64) for k in ("q", "dq", "act", "l_m", "v_m", "f_m", "t")]
        ints = np.ascontiguousarray(s["ints"], dtype=np.int32)
        self.lib.ref_set_state(self.h, *[_ptr(a, _dp) for a in arrs], _ptr(ints, _ip))

    def get_sampler(self):
        ema = np.zeros((self.n, self.bins))
        self.lib.ref_get_sampler(self.h, _ptr(ema, _dp))
        return ema

    def set_sampler(self, ema):
        e = np.ascontiguousarray(np.broadcast_to(ema, (self.n, self.bins)), dtype=np.float64)
        self.lib.ref_set_sampler(self.h, _ptr(e, _dp))

    def record_own_outcomes(self):
        self.lib.ref_record_own_outcomes(self.h)

    def drain_outcomes(self, cap=64):
        bins = np.zeros((self.n, cap), dtype=np.int32)
        failed = np.zeros((self.n, cap), dtype=np.uint8)
        counts = np.zeros(self.n, dtype=np.int32)
        self.lib.ref_drain_outcomes(self.h, _ptr(bins, _ip), _ptr(failed, _up), _ptr(counts, _ip), cap)
        return bins, failed, counts

    def rng_raw(self, env, n):
        out = np.zeros(n, dtype=np.uint64)
        self.lib.ref_rng_raw(self.h, env, n, out.ctypes.data_as(C.POINTER(C.c_uint64)))
        return out

    def rng_serialize(self, env):
        """The reference's own Rng::serialize() of env `env` (rng.hpp:56-61)."""
        buf = C.create_string_buffer(16384)
        n = self.lib.ref_rng_serialize(self.h, int(env), buf, len(buf))
        assert n < len(buf)
        return buf.value.decode()

    def rng_deserialize(self, env, text):
        self.lib.ref_rng_deserialize(self.h, int(env), text.encode())

    def set_discriminator(self, theta, hidden):
        """ref_bench's tracking reward: the reference's Mlp(dΔ, hidden, 1, Sigmoid) with theta."""
        theta = np.ascontiguousarray(theta, dtype=np.float64)
        rc = self.lib.ref_set_discriminator(self.h, _ptr(theta, _dp), theta.size, hidden)
        if rc != 0:
            raise ValueError("ref_set_discriminator: parameter count mismatch")

    def bench(self, steps, action_seed=0x5EED):
        n = C.c_int64(0)
        secs = self.lib.ref_bench(self.h, steps, C.c_uint64(action_seed), C.byref(n))
        return secs, int(n.value)

    # model-level functions
    def mass_matrix(self, q):
        q = np.ascontiguousarray(q, dtype=np.float64)
        M = np.zeros((self.nq, self.nq))
        self.lib.ref_mass_matrix(self.h, _ptr(q, _dp), _ptr(M, _dp))
        return M

    def moment_arms(self, q):
        q = np.ascontiguousarray(q, dtype=np.float64)
        J = np.zeros((self.nm, self.nq))
        self.lib.ref_moment_arms(self.h, _ptr(q, _dp), _ptr(J, _dp))
        return J

    def bias_forces(self, q, dq):
        q = np.ascontiguousarray(q, dtype=np.float64)
        dq = np.ascontiguousarray(dq, dtype=np.float64)
        c = np.zeros(self.nq)
        self.lib.ref_bias_forces(self.h, _ptr(q, _dp), _ptr(dq, _dp), _ptr(c, _dp))
        return c

    def mtu_length(self, q, m):
        q = np.ascontiguousarray(q, dtype=np.float64)
        return self.lib.ref_mtu_length(self.h, _ptr(q, _dp), m)

    def mechanical_energy(self, q, dq):
        q = np.ascontiguousarray(q, dtype=np.float64)
        dq = np.ascontiguousarray(dq, dtype=np.float64)
        return self.lib.ref_mechanical_energy(self.h, _ptr(q, _dp), _ptr(dq, _dp))

    def key_bodies(self, q):
        q = np.ascontiguousarray(q, dtype=np.float64)
        pos = np.zeros((self.nk, 2))
        ang = np.zeros(self.nk)
        self.lib.ref_key_bodies(self.h, _ptr(q, _dp), _ptr(pos, _dp), _ptr(ang, _dp))
        return pos, ang


def rng_uniform(seed, lo, hi, n):
    """n draws of the reference's msk::Rng(seed).uniform(lo, hi) (rng.hpp:26-30)."""
    out = np.zeros(n)
    ref_lib().ref_rng_uniform(C.c_uint64(seed), float(lo), float(hi), int(n), out.ctypes.data_as(_dp))
    return out


# ---- the reference's nn.cpp (Mlp / Adam / RunningNorm), nn.cpp:16-284 ----------
HEAD_LINEAR, HEAD_SIGMOID, HEAD_AFFINE = 0, 1, 2


def _d(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(_dp)


def ref_mlp_init(n_in, hidden, n_out, seed, final_init_scale=1.0):
    L = ref_lib()
    n = L.ref_mlp_init(n_in, hidden, n_out, C.c_uint64(seed), final_init_scale, None)
    th = np.zeros(n)
    L.ref_mlp_init(n_in, hidden, n_out, C.c_uint64(seed), final_init_scale, th.ctypes.data_as(_dp))
    return th


def ref_mlp_forward(theta, n_in, hidden, n_out, X, head=HEAD_SIGMOID, affine=(1.0, 0.0)):
    th, pth = _d(theta)
    x, px = _d(np.atleast_2d(X))
    y = np.zeros((x.shape[0], n_out))
    ref_lib().ref_mlp_forward(pth, th.size, n_in, hidden, n_out, head, affine[0], affine[1], px, x.shape[0],
                              y.ctypes.data_as(_dp))
    return y


def ref_mlp_backward(theta, n_in, hidden, n_out, X, upstream, head=HEAD_SIGMOID, affine=(1.0, 0.0)):
    """(grad [n], input_grad [B x in]) of Mlp::backward from a zero gradient."""
    th, pth = _d(theta)
    x, px = _d(np.atleast_2d(X))
    up, pup = _d(np.atleast_2d(upstream))
    g = np.zeros(th.size)
    ig = np.zeros(x.shape)
    ref_lib().ref_mlp_backward(pth, th.size, n_in, hidden, n_out, head, affine[0], affine[1], px, x.shape[0], pup,
                               g.ctypes.data_as(_dp), ig.ctypes.data_as(_dp))
    return g, ig


def ref_mlp_gp_backward(theta, n_in, hidden, X, head=HEAD_SIGMOID):
    """(grad [n], penalty [B]) of Mlp::gradient_penalty_backward from a zero gradient."""
    th, pth = _d(theta)
    x, px = _d(np.atleast_2d(X))
    g = np.zeros(th.size)
    pen = np.zeros(x.shape[0])
    ref_lib().ref_mlp_gp_backward(pth, th.size, n_in, hidden, head, px, x.shape[0], g.ctypes.data_as(_dp),
                                  pen.ctypes.data_as(_dp))
    return g, pen


class RefAdam:
    """Adam::step (nn.cpp:224-240) with the state held here."""

    def __init__(self, n, lr):
        self.lr, self.m, self.v = lr, np.zeros(n), np.zeros(n)
        self.step_count, self.skipped = C.c_int64(0), C.c_int64(0)

    def step(self, params, grad):
        g, pg = _d(grad)
        ok = ref_lib().ref_adam_step(params.ctypes.data_as(_dp), pg, params.size, self.lr, self.m.ctypes.data_as(_dp),
                                     self.v.ctypes.data_as(_dp), C.byref(self.step_count), C.byref(self.skipped))
        return bool(ok)


def ref_running_norm(X, count, mean, var):
    """RunningNorm::update(X) then apply(X) (nn.cpp:246-277): (count, mean, var, Y)."""
    x, px = _d(np.atleast_2d(X))
    c = np.array([count], dtype=np.float64)
    m = np.array(mean, dtype=np.float64)
    v = np.array(var, dtype=np.float64)
    y = np.zeros(x.shape)
    ref_lib().ref_running_norm(px, x.shape[0], x.shape[1], c.ctypes.data_as(_dp), m.ctypes.data_as(_dp),
                               v.ctypes.data_as(_dp), y.ctypes.data_as(_dp))
    return float(c[0]), m, v, y
