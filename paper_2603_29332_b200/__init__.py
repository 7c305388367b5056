"""B200-native batched musculoskeletal env-stepper (host mirror of msk::Env).

The product is the sm_100a shared library ``libmsk_b200.so`` with the C ABI in
``include/msk_gpu.h``.  This module binds that ABI with ctypes and exposes the
reference's environment verbs (``/root/reference/proj/include/msk/env.hpp:86-145``)
in batched form over torch CUDA tensors — torch is used for device memory
and streams only.  There is no CPU fallback: importing works anywhere, but
creating an :class:`EnvBatch` needs the library and a B200, and fails loudly
otherwise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

__all__ = ["EnvConfig", "RewardConfig", "RewardMode", "EnvBatch", "lib", "LIB_PATH", "MskError", "mlp_init", "Policy", "Rollout",
           "FLAG_DONE", "FLAG_FAILED", "FLAG_DIVERGED", "FLAG_NOT_STEPPED", "FLAG_BAD_ACTION"]

LIB_PATH = os.environ.get("MSK_B200_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libmsk_b200.so")

FLAG_DONE, FLAG_FAILED, FLAG_DIVERGED, FLAG_NOT_STEPPED, FLAG_BAD_ACTION = 1, 2, 4, 8, 16


def mlp_init(n_in, hidden, seed, n_out=1, final_init_scale=1.0):
    """Mlp(MlpShape{n_in, hidden, n_out}, seed) flat f64 parameters (nn.cpp:16-38)."""
    import numpy as np

    n = lib().msk_mlp_param_count(n_in, hidden, n_out)
    if n < 0:
        raise ValueError("bad Mlp shape")
    theta = np.zeros(n)
    rc = lib().msk_mlp_init(theta.ctypes.data, n_in, hidden, n_out, C.c_uint64(seed), float(final_init_scale))
    if rc != 0:
        raise MskError(rc, lib().msk_gpu_last_error(None).decode())
    return theta


class Policy:
    """On-device policy sampling (msk_policy_*): Gaussian π⁽⁰⁾ + flow-ODE ψ on the tensor cores.

    pi_theta: Mlp(obs_dim, hidden, n_actions) flat f64 params; psi_theta: Mlp(5 + obs_dim +
    n_actions, hidden, n_actions); log_std [n_actions]; head y = head_scale * z + head_offset."""

    TIME_FEATURES = 5

    def __init__(self, obs_dim, n_actions, hidden, pi_theta, log_std, psi_theta, n_ode=20, dt_ode=0.05,
                 max_envs=4096, head_scale=1.0, head_offset=0.0, device=None):
        import numpy as np
        import torch

        self.torch = torch
        device = torch.cuda.current_device() if device is None else device
        self.obs_dim, self.nm, self.hidden, self.n_ode, self.dt = obs_dim, n_actions, hidden, n_ode, dt_ode
        self.max_envs = max_envs
        self.device = torch.device("cuda", device)
        self._keep = [np.ascontiguousarray(np.asarray(x, dtype=np.float64)) for x in (pi_theta, log_std, psi_theta)]
        pi, ls, psi = self._keep
        h = C.c_void_p()
        rc = lib().msk_policy_create(obs_dim, n_actions, hidden, pi.ctypes.data, pi.size, head_scale, head_offset,
                                     ls.ctypes.data, psi.ctypes.data, psi.size, n_ode, dt_ode, max_envs, device,
                                     C.byref(h))
        if rc != 0:
            raise MskError(rc, lib().msk_policy_last_error(None).decode())
        self.h = h

    def _ck(self, rc):
        if rc != 0:
            raise MskError(rc, lib().msk_policy_last_error(self.h).decode())

    def set_norm(self, mean, var, count):
        import numpy as np

        if mean is None or var is None or count == 0:  # RunningNorm with count 0: identity
            self._ck(lib().msk_policy_set_norm(self.h, None, None, 0.0))
            return
        m = np.ascontiguousarray(mean, dtype=np.float64)
        v = np.ascontiguousarray(var, dtype=np.float64)
        self._ck(lib().msk_policy_set_norm(self.h, m.ctypes.data, v.ctypes.data, float(count)))

    def sample(self, obs, explore=False, seed=0, step=0, global_env_offset=0, actions=None, a0=None, logprob=None,
               graph=False, stream=None):
        """Returns actions [n x n_actions] (device); a0 / logprob filled when given."""
        torch = self.torch
        n = obs.shape[0]
        actions = actions if actions is not None else torch.empty(n, self.nm, device=self.device)
        fn = lib().msk_policy_sample_graph if graph else lib().msk_policy_sample
        s = stream.cuda_stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
        self._ck(fn(self.h, _p(obs.contiguous()), n, int(bool(explore)), C.c_uint64(seed), C.c_uint32(step),
                    int(global_env_offset), _p(actions), _p(a0), _p(logprob), s))
        return actions

    def close(self):
        if getattr(self, "h", None):
            lib().msk_policy_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Rollout:
    """On-device rollout buffer (h x E, step-major) + GAE (msk_rollout_*)."""

    def __init__(self, n_envs, horizon, obs_dim, act_dim, delta_dim, device=None):
        import torch

        self.torch = torch
        device = torch.cuda.current_device() if device is None else device
        self.E, self.h = n_envs, horizon
        h = C.c_void_p()
        rc = lib().msk_rollout_create(n_envs, horizon, obs_dim, act_dim, delta_dim, device, C.byref(h))
        if rc != 0:
            raise MskError(rc, lib().msk_rollout_last_error(None).decode())
        self.h_ = h
        self.device = torch.device("cuda", device)

    def _ck(self, rc):
        if rc != 0:
            raise MskError(rc, lib().msk_rollout_last_error(self.h_).decode())

    def record(self, t, obs=None, a0=None, actions=None, logprob=None, reward=None, flags=None, value=None,
               delta=None, stream=None):
        s = stream.cuda_stream if stream is not None else self.torch.cuda.current_stream(self.device).cuda_stream
        self._ck(lib().msk_rollout_record(self.h_, int(t), _p(obs), _p(a0), _p(actions), _p(logprob), _p(reward),
                                          _p(flags), _p(value), _p(delta), s))

    def gae(self, bootstrap_value, gamma=0.99, lam=0.95, normalize=True, stream=None):
        """(advantages, returns), each [h x E] float32 on the device."""
        torch = self.torch
        adv = torch.empty(self.h, self.E, device=self.device)
        ret = torch.empty(self.h, self.E, device=self.device)
        s = stream.cuda_stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
        self._ck(lib().msk_rollout_gae(self.h_, _p(bootstrap_value.contiguous()), float(gamma), float(lam),
                                       int(bool(normalize)), _p(adv), _p(ret), s))
        return adv, ret

    def minibatch(self, seed, epoch, index, mb_size, obs_dim, act_dim, stream=None):
        """PPO minibatch `index` of epoch `epoch` (msk_rollout_minibatch): dict of
        device tensors obs, a0, actions, logprob, advantages, returns, value, record_ids."""
        torch = self.torch
        n = self.h * self.E
        rows = max(0, min(mb_size, n - index * mb_size))
        f = lambda *shape: torch.empty(*shape, device=self.device)  # noqa: E731
        out = dict(obs=f(rows, obs_dim), a0=f(rows, act_dim), actions=f(rows, act_dim), logprob=f(rows),
                   advantages=f(rows), returns=f(rows), value=f(rows),
                   record_ids=torch.empty(rows, dtype=torch.int32, device=self.device))
        s = stream.cuda_stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
        self._ck(lib().msk_rollout_minibatch(self.h_, C.c_uint64(seed), int(epoch), int(index), int(mb_size),
                                             *[_p(out[k]) for k in ("obs", "a0", "actions", "logprob", "advantages",
                                                                   "returns", "value", "record_ids")], s))
        return out

    def field(self, index, cols, dtype=None):
        """Device tensor view [h * E x cols] of a stored field (msk_rollout_field:
        0 obs, 1 a0, 2 actions, 3 logprob, 4 reward, 5 done, 6 value, 7 delta)."""
        torch = self.torch
        dtype = dtype or torch.float32
        ptr = lib().msk_rollout_field(self.h_, int(index))
        n = self.h * self.E * cols
        return _wrap_device(ptr, n, dtype, self.device).view(self.h * self.E, cols)

    def close(self):
        if getattr(self, "h_", None):
            lib().msk_rollout_destroy(self.h_)
            self.h_ = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DiscTrainer:
    """Discriminator training step on the device (msk_disc_trainer_*; SPEC.md:412-421
    train_discriminator): one Adam step (nn.cpp:224-240) on
    -log clamp(D(0)) - mean log(1 - clamp(D(Δ))) + λ mean ||∇_Δ D(Δ)||².
    math: 0 fp32-class (split-bf16 tcgen05 GEMMs, 3 MMAs per product), 1 bf16 tcgen05 GEMMs."""

    def __init__(self, n_in, hidden, theta, lr=3e-5, grad_penalty=10.0, max_rows=4096, math=0, device=None):
        import numpy as np
        import torch

        self.torch = torch
        device = torch.cuda.current_device() if device is None else device
        theta = np.ascontiguousarray(theta, dtype=np.float64)
        self.n_in, self.hidden, self.n_params = n_in, hidden, len(theta)
        h = C.c_void_p()
        rc = lib().msk_disc_trainer_create(n_in, hidden, theta.ctypes.data, len(theta), float(lr),
                                           float(grad_penalty), int(max_rows), int(math), device, C.byref(h))
        if rc != 0:
            raise MskError(rc, lib().msk_disc_trainer_last_error(None).decode())
        self.h_ = h
        self.device = torch.device("cuda", device)
        self.loss = torch.zeros(3, dtype=torch.float64, device=self.device)

    def _ck(self, rc):
        if rc != 0:
            raise MskError(rc, lib().msk_disc_trainer_last_error(self.h_).decode())

    def _s(self, stream):
        return stream.cuda_stream if stream is not None else self.torch.cuda.current_stream(self.device).cuda_stream

    def step(self, delta, stream=None):
        """One update on delta [rows x ld] (f32, device); returns the device loss
        tensor {total, logistic, mean penalty} at the pre-step parameters."""
        self._ck(lib().msk_disc_train_step(self.h_, _p(delta), delta.shape[0], delta.stride(0), _p(self.loss),
                                           self._s(stream)))
        return self.loss

    def gradient(self, delta, stream=None):
        """(grad [n_params] f32, loss [3] f64) at the current parameters, no update."""
        g = self.torch.empty(self.n_params, dtype=self.torch.float32, device=self.device)
        self._ck(lib().msk_disc_trainer_gradient(self.h_, _p(delta), delta.shape[0], delta.stride(0), _p(g),
                                                 _p(self.loss), self._s(stream)))
        return g, self.loss

    def params(self):
        """(theta f64 numpy, adam_steps, adam_skipped); synchronises."""
        import numpy as np

        th = np.zeros(self.n_params)
        st, sk = C.c_int64(), C.c_int64()
        self._ck(lib().msk_disc_trainer_get_params(self.h_, th.ctypes.data, C.byref(st), C.byref(sk)))
        return th, st.value, sk.value

    def publish(self, env, stream=None):
        """Refresh env's reward discriminator from this trainer's θ on the device."""
        env._ck(lib().msk_disc_trainer_publish(self.h_, env.h, self._s(stream)))

    def close(self):
        if getattr(self, "h_", None):
            lib().msk_disc_trainer_destroy(self.h_)
            self.h_ = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _wrap_device(ptr, n, dtype, device):
    """A torch tensor viewing n elements of library-owned device memory (no copy)."""
    import torch

    class _Arr:  # __cuda_array_interface__ v3
        pass

    typestr = {torch.float32: "<f4", torch.uint8: "|u1", torch.float64: "<f8", torch.int32: "<i4"}[dtype]
    a = _Arr()
    a.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (int(ptr), False), "version": 3,
                                  "strides": None}
    return torch.as_tensor(a, device=device)


def time_features(t):
    import numpy as np

    out = np.zeros(5)
    lib().msk_policy_time_features(float(t), out.ctypes.data)
    return out


class MskError(RuntimeError):
    """A non-zero msk_status from the C ABI (1 = contract/config, 3 = CUDA)."""

    def __init__(self, code, msg):
        super().__init__(f"[msk status {code}] {msg}")
        self.code = code


class RewardMode:
    """msk::RewardMode (env.hpp:30)."""
    ImitationOnly, ImitationEmg, ImitationPower = 0, 1, 2


@dataclass
class EnvConfig:
    """msk::EnvConfig defaults (env.hpp:39-47)."""
    episode_horizon: int = 250
    rsi: bool = True
    adaptive_bins: int = 10
    adaptive_mix: float = 0.2
    adaptive_decay: float = 0.99
    termination_body_err: float = 0.5
    init_activation: float = 0.01


@dataclass
class RewardConfig:
    """msk::RewardConfig defaults (env.hpp:32-37)."""
    mode: int = RewardMode.ImitationOnly
    w_emg: float = 100.0
    w_power: float = 0.05
    emg_channel_map: list = field(default_factory=list)


class _EnvConfigC(C.Structure):
    _fields_ = [("episode_horizon", C.c_int32), ("rsi", C.c_int32), ("adaptive_bins", C.c_int32),
                ("pad0", C.c_int32), ("adaptive_mix", C.c_double), ("adaptive_decay", C.c_double),
                ("termination_body_err", C.c_double), ("init_activation", C.c_double)]


class _RewardConfigC(C.Structure):
    _fields_ = [("mode", C.c_int32), ("n_emg_channels", C.c_int32), ("w_emg", C.c_double),
                ("w_power", C.c_double), ("emg_channel_map", C.POINTER(C.c_int32))]


class _Dims(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("n_envs", "nq", "n_muscles", "obs_dim", "delta_dim", "n_links",
                                          "n_joints", "n_key", "n_spheres", "frames", "floating",
                                          "adaptive_bins")]


_LIB = None
_vp = C.c_void_p


def lib():
    """Loads libmsk_b200.so (raises if it was not built — there is no fallback)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                              f"g.build()'` (make -C paper_2603_29332_b200/csrc)")
        L = C.CDLL(LIB_PATH)
        L.msk_gpu_create.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(_EnvConfigC), C.POINTER(_RewardConfigC),
                                     C.c_int32, C.c_uint64, C.c_int64, C.c_int, C.POINTER(_vp)]
        L.msk_gpu_destroy.argtypes = [_vp]
        L.msk_gpu_last_error.restype = C.c_char_p
        L.msk_gpu_last_error.argtypes = [_vp]
        L.msk_gpu_dims.argtypes = [_vp, C.POINTER(_Dims)]
        L.msk_gpu_set_eval_mode.argtypes = [_vp, C.c_int32]
        L.msk_gpu_reset.argtypes = [_vp, _vp, C.c_uint8, _vp, _vp, _vp]
        L.msk_gpu_reset_to_frame.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp]
        L.msk_gpu_step.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
        L.msk_gpu_step_host.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp]
        L.msk_gpu_step_host_rewarded.argtypes = [_vp] * 7
        L.msk_gpu_step_host_async.argtypes = [_vp] * 7
        L.msk_gpu_host_wait.argtypes = [_vp]
        L.msk_gpu_set_host_pipeline.argtypes = [_vp, C.c_int32, C.c_int32]
        L.msk_gpu_rollout_stats.argtypes = [_vp] * 5
        L.msk_policy_create.argtypes = [C.c_int32, C.c_int32, C.c_int32, _vp, C.c_int64, C.c_double, C.c_double, _vp,
                                        _vp, C.c_int64, C.c_int32, C.c_double, C.c_int32, C.c_int32, _vp]
        L.msk_policy_destroy.argtypes = [_vp]
        L.msk_policy_last_error.restype = C.c_char_p
        L.msk_policy_last_error.argtypes = [_vp]
        L.msk_policy_set_norm.argtypes = [_vp, _vp, _vp, C.c_double]
        L.msk_policy_sample.argtypes = [_vp, _vp, C.c_int32, C.c_int32, C.c_uint64, C.c_uint32, C.c_int64, _vp, _vp,
                                        _vp, _vp]
        L.msk_policy_sample_graph.argtypes = L.msk_policy_sample.argtypes
        L.msk_policy_time_features.restype = C.c_int32
        L.msk_policy_time_features.argtypes = [C.c_double, _vp]
        L.msk_gemm_test.argtypes = [_vp, C.c_int32, C.c_int32, _vp, _vp, C.c_int32, C.c_int32, _vp]
        L.msk_rollout_create.argtypes = [C.c_int32] * 6 + [_vp]
        L.msk_rollout_destroy.argtypes = [_vp]
        L.msk_rollout_last_error.restype = C.c_char_p
        L.msk_rollout_last_error.argtypes = [_vp]
        L.msk_rollout_record.argtypes = [_vp, C.c_int32] + [_vp] * 9
        L.msk_rollout_gae.argtypes = [_vp, _vp, C.c_float, C.c_float, C.c_int32, _vp, _vp, _vp]
        L.msk_rollout_minibatch.argtypes = [_vp, C.c_uint64, C.c_int32, C.c_int32, C.c_int32] + [_vp] * 9
        L.msk_rollout_field.restype = C.c_void_p
        L.msk_rollout_field.argtypes = [_vp, C.c_int32]
        L.msk_gpu_obs_moments.argtypes = [_vp, _vp, C.c_int32, _vp, _vp]
        L.msk_gpu_obs_moments_fold.argtypes = [_vp, _vp, C.c_int32, _vp, _vp]
        L.msk_gpu_iteration_exchange.argtypes = [_vp, _vp, C.c_int32, _vp, _vp, _vp, _vp, _vp]
        L.msk_gpu_set_discriminator.argtypes = [_vp, _vp, C.c_int64, C.c_int32]
        L.msk_gpu_set_discriminator_mode.argtypes = [_vp, C.c_int32]
        L.msk_mlp_param_count.restype = C.c_int64
        L.msk_mlp_param_count.argtypes = [C.c_int32, C.c_int32, C.c_int32]
        L.msk_mlp_init.argtypes = [_vp, C.c_int32, C.c_int32, C.c_int32, C.c_uint64, C.c_double]
        L.msk_gpu_clear_discriminator.argtypes = [_vp]
        L.msk_gpu_discriminator_reward.argtypes = [_vp, _vp, C.c_int32, _vp, _vp]
        L.msk_gpu_step_rewarded.argtypes = [_vp] * 10
        L.msk_gpu_observe.argtypes = [_vp, _vp, _vp]
        L.msk_gpu_tracking_error.argtypes = [_vp, _vp, _vp]
        L.msk_gpu_force_state_to_reference.argtypes = [_vp, _vp]
        L.msk_gpu_get_state.argtypes = [_vp] + [_vp] * 8 + [_vp]
        L.msk_gpu_set_state.argtypes = [_vp] + [_vp] * 8 + [_vp]
        L.msk_gpu_get_sampler.argtypes = [_vp, _vp, _vp]
        L.msk_gpu_set_sampler.argtypes = [_vp, _vp, C.c_int32, _vp]
        L.msk_gpu_drain_outcomes.argtypes = [_vp, _vp, _vp, _vp, C.c_int32, _vp]
        L.msk_gpu_record_own_outcomes.argtypes = [_vp, _vp]
        L.msk_gpu_merge_outcomes.argtypes = [_vp, _vp, _vp, _vp, C.c_int64, C.c_int32, _vp]
        L.msk_gpu_rng_raw.argtypes = [_vp, C.c_int32, C.c_int32, _vp, _vp]
        L.msk_gpu_get_rng.argtypes = [_vp, _vp, _vp, _vp]
        L.msk_gpu_substeps.argtypes = [_vp, _vp, C.c_int32, _vp, _vp, _vp]
        L.msk_gpu_set_rng.argtypes = [_vp, _vp, _vp, _vp]
        L.msk_gpu_set_outcome_capacity.argtypes = [_vp, C.c_int32, _vp]
        L.msk_gpu_outcomes_dropped.argtypes = [_vp, C.POINTER(C.c_int64)]
        L.msk_gpu_fill_excitations.argtypes = [_vp, C.c_uint64, C.c_uint32, _vp, _vp]
        L.msk_gpu_launch_count.restype = C.c_int64
        L.msk_disc_trainer_create.argtypes = [C.c_int32, C.c_int32, _vp, C.c_int64, C.c_double, C.c_double,
                                              C.c_int32, C.c_int32, C.c_int32, _vp]
        L.msk_disc_trainer_destroy.argtypes = [_vp]
        L.msk_disc_trainer_last_error.restype = C.c_char_p
        L.msk_disc_trainer_last_error.argtypes = [_vp]
        L.msk_disc_train_step.argtypes = [_vp, _vp, C.c_int32, C.c_int32, _vp, _vp]
        L.msk_disc_trainer_gradient.argtypes = [_vp, _vp, C.c_int32, C.c_int32, _vp, _vp, _vp]
        L.msk_disc_trainer_get_params.argtypes = [_vp, _vp, _vp, _vp]
        L.msk_disc_trainer_publish.argtypes = [_vp, _vp, _vp]
        L.msk_gpu_launch_count.argtypes = [_vp]
        for name in ("msk_gpu_create", "msk_gpu_dims", "msk_gpu_set_eval_mode", "msk_gpu_reset",
                     "msk_gpu_reset_to_frame", "msk_gpu_step", "msk_gpu_step_host", "msk_gpu_observe",
                     "msk_gpu_tracking_error", "msk_gpu_force_state_to_reference", "msk_gpu_get_state",
                     "msk_gpu_set_state", "msk_gpu_get_sampler", "msk_gpu_set_sampler", "msk_gpu_drain_outcomes",
                     "msk_gpu_record_own_outcomes", "msk_gpu_merge_outcomes", "msk_gpu_rng_raw",
                     "msk_gpu_fill_excitations", "msk_gpu_get_rng", "msk_gpu_set_rng",
                     "msk_gpu_set_outcome_capacity", "msk_gpu_outcomes_dropped", "msk_gpu_substeps"):
            getattr(L, name).restype = C.c_int
        _LIB = L
    return _LIB


def _p(t):
    return None if t is None else C.c_void_p(t.data_ptr())


class EnvBatch:
    """E environments on one GPU with the verbs of ``msk::Env``.

    Buffers are torch CUDA tensors; every call is asynchronous on the current
    torch stream (or ``stream``).  Env e's seed is ``base_seed +
    global_env_offset + e`` (``Env(seed)``, env.cpp:74-76).
    """

    def __init__(self, model_path, clip_path, n_envs, cfg: EnvConfig | None = None,
                 reward: RewardConfig | None = None, base_seed=0x5EED, global_env_offset=0, device=None):
        import torch

        self.torch = torch
        cfg = cfg or EnvConfig()
        reward = reward or RewardConfig()
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", device)
        ec = _EnvConfigC(int(cfg.episode_horizon), int(bool(cfg.rsi)), int(cfg.adaptive_bins), 0,
                         float(cfg.adaptive_mix), float(cfg.adaptive_decay), float(cfg.termination_body_err),
                         float(cfg.init_activation))
        self._emg = (C.c_int32 * max(1, len(reward.emg_channel_map)))(*reward.emg_channel_map)
        rc = _RewardConfigC(int(reward.mode), len(reward.emg_channel_map), float(reward.w_emg),
                            float(reward.w_power), self._emg)
        L = lib()
        h = _vp()
        rcode = L.msk_gpu_create(os.fsencode(model_path), os.fsencode(clip_path), C.byref(ec), C.byref(rc),
                                 int(n_envs), C.c_uint64(base_seed), int(global_env_offset), int(device), C.byref(h))
        if rcode != 0:
            raise MskError(rcode, L.msk_gpu_last_error(None).decode())
        self.h = h
        d = _Dims()
        L.msk_gpu_dims(h, C.byref(d))
        self.n = d.n_envs
        self.nq, self.nm, self.obs_dim, self.delta_dim = d.nq, d.n_muscles, d.obs_dim, d.delta_dim
        self.n_links, self.nj, self.nk, self.n_spheres = d.n_links, d.n_joints, d.n_key, d.n_spheres
        self.frames, self.floating, self.bins = d.frames, bool(d.floating), d.adaptive_bins
        self.cfg, self.reward = cfg, reward

    # -- plumbing ---------------------------------------------------------------
    def _s(self, stream):
        s = stream if stream is not None else self.torch.cuda.current_stream(self.device)
        return C.c_void_p(s.cuda_stream)

    def _ck(self, rcode):
        if rcode != 0:
            raise MskError(rcode, lib().msk_gpu_last_error(self.h).decode())

    def _empty(self, *shape, dtype=None):
        return self.torch.empty(*shape, dtype=dtype or self.torch.float32, device=self.device)

    def close(self):
        if getattr(self, "h", None):
            lib().msk_gpu_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launch_count(self):
        return int(lib().msk_gpu_launch_count(self.h))

    # -- Env verbs (env.hpp:86-123) ---------------------------------------------
    def set_eval_mode(self, eval_mode=True):
        self._ck(lib().msk_gpu_set_eval_mode(self.h, int(bool(eval_mode))))

    def reset(self, mask=None, mask_bits=0xFF, obs=None, start_frames=None, stream=None):
        """Env::reset for envs with ``mask & mask_bits`` (all when mask is None)."""
        obs = obs if obs is not None else self._empty(self.n, self.obs_dim)
        self._ck(lib().msk_gpu_reset(self.h, _p(mask), int(mask_bits), _p(obs), _p(start_frames), self._s(stream)))
        return obs

    def reset_to_frame(self, frames, mask=None, obs=None, stream=None):
        torch = self.torch
        fr = torch.as_tensor(frames, dtype=torch.int32, device=self.device).expand(self.n).contiguous()
        obs = obs if obs is not None else self._empty(self.n, self.obs_dim)
        bad = self._empty(self.n, dtype=torch.uint8)
        self._ck(lib().msk_gpu_reset_to_frame(self.h, _p(fr), _p(mask), _p(obs), _p(bad), self._s(stream)))
        return obs, bad

    def set_discriminator(self, theta, hidden):
        """Load D = Mlp(delta_dim, hidden, 1, Sigmoid) from its flat f64 parameters (nn.cpp layout)."""
        import numpy as np

        th = np.ascontiguousarray(np.asarray(theta, dtype=np.float64))
        self._ck(lib().msk_gpu_set_discriminator(self.h, th.ctypes.data, th.size, int(hidden)))
        self._disc = True

    def set_discriminator_mode(self, fast):
        """False (default): fp32-class split-bf16 operands; True: bf16 operands (fast)."""
        self._ck(lib().msk_gpu_set_discriminator_mode(self.h, 1 if fast else 0))

    def clear_discriminator(self):
        self._ck(lib().msk_gpu_clear_discriminator(self.h))
        self._disc = False

    def discriminator_reward(self, delta, reward=None, stream=None):
        """r = -log(1 - clamp(D(delta), 1e-4, 1 - 1e-4)) per row of delta [n x delta_dim] (device)."""
        d = delta if delta.dtype == self.torch.float32 and delta.is_contiguous() else delta.float().contiguous()
        n = d.shape[0]
        reward = reward if reward is not None else self._empty(n)
        self._ck(lib().msk_gpu_discriminator_reward(self.h, _p(d), n, _p(reward), self._s(stream)))
        return reward

    def step(self, actions, obs=None, delta=None, reward_aux=None, flags=None, muscle_power=None,
             contact_force=None, want_power=False, want_contact=False, stream=None, reward=None,
             want_reward=False):
        """Env::step for every env; returns a dict of [E x ...] tensors (StepResult fields).
        With want_reward / reward (and a discriminator set): Env::step(action, fn),
        reward = r(D(delta)) + reward_aux."""
        torch = self.torch
        a = actions if actions.dtype == torch.float32 and actions.is_contiguous() else actions.float().contiguous()
        out = dict(
            obs=obs if obs is not None else self._empty(self.n, self.obs_dim),
            delta=delta if delta is not None else self._empty(self.n, self.delta_dim),
            reward_aux=reward_aux if reward_aux is not None else self._empty(self.n),
            flags=flags if flags is not None else self._empty(self.n, dtype=torch.uint8),
        )
        if want_power or muscle_power is not None:
            out["muscle_power"] = muscle_power if muscle_power is not None else self._empty(self.n, self.nm)
        if want_contact or contact_force is not None:
            out["contact_force"] = contact_force if contact_force is not None else self._empty(self.n, self.n_links, 2)
        if want_reward or reward is not None:
            out["reward"] = reward if reward is not None else self._empty(self.n)
            self._ck(lib().msk_gpu_step_rewarded(self.h, _p(a), _p(out["obs"]), _p(out["delta"]), _p(out["reward"]),
                                                 _p(out["reward_aux"]), _p(out["flags"]),
                                                 _p(out.get("muscle_power")), _p(out.get("contact_force")),
                                                 self._s(stream)))
            return out
        self._ck(lib().msk_gpu_step(self.h, _p(a), _p(out["obs"]), _p(out["delta"]), _p(out["reward_aux"]),
                                    _p(out["flags"]), _p(out.get("muscle_power")), _p(out.get("contact_force")),
                                    self._s(stream)))
        return out

    def step_host(self, actions_host, obs_host=None, delta_host=None, reward_aux_host=None, flags_host=None,
                  reward_host=None):
        """Env::step with HOST (ideally pinned) tensors; synchronous, pipelined H2D/kernel/D2H.
        With reward_host (and a discriminator set): Env::step(action, fn)."""
        if reward_host is not None:
            self._ck(lib().msk_gpu_step_host_rewarded(self.h, _p(actions_host), _p(obs_host), _p(delta_host),
                                                      _p(reward_host), _p(reward_aux_host), _p(flags_host)))
            return
        self._ck(lib().msk_gpu_step_host(self.h, _p(actions_host), _p(obs_host), _p(delta_host),
                                         _p(reward_aux_host), _p(flags_host)))

    def step_host_async(self, actions_host, obs_host=None, delta_host=None, reward_aux_host=None, flags_host=None,
                        reward_host=None):
        """Enqueue a host-buffer step and return; pair with host_wait() (buffers must be pinned)."""
        self._ck(lib().msk_gpu_step_host_async(self.h, _p(actions_host), _p(obs_host), _p(delta_host),
                                               _p(reward_host), _p(reward_aux_host), _p(flags_host)))

    def host_wait(self):
        self._ck(lib().msk_gpu_host_wait(self.h))

    def set_host_pipeline(self, chunks, streams):
        """Env chunks and streams of the host-buffer pipeline."""
        self._ck(lib().msk_gpu_set_host_pipeline(self.h, int(chunks), int(streams)))

    def observe(self, obs=None, stream=None):
        obs = obs if obs is not None else self._empty(self.n, self.obs_dim)
        self._ck(lib().msk_gpu_observe(self.h, _p(obs), self._s(stream)))
        return obs

    def tracking_error(self, delta=None, stream=None):
        delta = delta if delta is not None else self._empty(self.n, self.delta_dim)
        self._ck(lib().msk_gpu_tracking_error(self.h, _p(delta), self._s(stream)))
        return delta

    def force_state_to_reference(self, stream=None):
        self._ck(lib().msk_gpu_force_state_to_reference(self.h, self._s(stream)))

    def get_state(self, stream=None):
        torch = self.torch
        n, nq, nm = self.n, self.nq, self.nm
        s = dict(q=self._empty(n, nq, dtype=torch.float64), dq=self._empty(n, nq, dtype=torch.float64),
                 act=self._empty(n, nm), l_m=self._empty(n, nm, dtype=torch.float64), v_m=self._empty(n, nm),
                 f_m=self._empty(n, nm),
                 t=self._empty(n, dtype=torch.float64), ints=self._empty(n, 4, dtype=torch.int32))
        self._ck(lib().msk_gpu_get_state(self.h, *[_p(s[k]) for k in ("q", "dq", "act", "l_m", "v_m", "f_m", "t",
                                                                      "ints")], self._s(stream)))
        return s

    def set_state(self, s, stream=None):
        torch = self.torch

        def cv(k, dt):
            if k not in s or s[k] is None:
                return None
            return torch.as_tensor(s[k], dtype=dt, device=self.device).contiguous()

        t = [cv("q", torch.float64), cv("dq", torch.float64), cv("act", torch.float32), cv("l_m", torch.float64),
             cv("v_m", torch.float32), cv("f_m", torch.float32), cv("t", torch.float64), cv("ints", torch.int32)]
        self._ck(lib().msk_gpu_set_state(self.h, *[_p(x) for x in t], self._s(stream)))
        self._keep = t

    def get_sampler(self, stream=None):
        ema = self._empty(self.n, self.bins, dtype=self.torch.float64)
        self._ck(lib().msk_gpu_get_sampler(self.h, _p(ema), self._s(stream)))
        return ema

    def set_sampler(self, ema, stream=None):
        torch = self.torch
        e = torch.as_tensor(ema, dtype=torch.float64, device=self.device).contiguous()
        bcast = int(e.dim() == 1)
        self._ck(lib().msk_gpu_set_sampler(self.h, _p(e), bcast, self._s(stream)))
        self._keep = e

    def drain_outcomes(self, cap=64, stream=None):
        torch = self.torch
        bins = self._empty(self.n, cap, dtype=torch.int32)
        failed = self._empty(self.n, cap, dtype=torch.uint8)
        counts = self._empty(self.n, dtype=torch.int32)
        self._ck(lib().msk_gpu_drain_outcomes(self.h, _p(bins), _p(failed), _p(counts), int(cap), self._s(stream)))
        return bins, failed, counts

    def record_own_outcomes(self, stream=None):
        self._ck(lib().msk_gpu_record_own_outcomes(self.h, self._s(stream)))

    def merge_outcomes(self, bins, failed, counts, stream=None):
        """Order-fixed merge of gathered outcome blocks (global env order) into one replicated sampler."""
        n_total, cap = bins.shape
        self._ck(lib().msk_gpu_merge_outcomes(self.h, _p(bins.contiguous()), _p(failed.contiguous()),
                                              _p(counts.contiguous()), int(n_total), int(cap), self._s(stream)))

    def rollout_stats(self, flags, stats, reward=None, stream=None):
        """stats[7] (f64, device) += this step's rollout statistics (see msk_gpu_rollout_stats)."""
        self._ck(lib().msk_gpu_rollout_stats(self.h, _p(reward), _p(flags), _p(stats), self._s(stream)))
        return stats

    def obs_moments(self, obs, out=None, stream=None):
        """[n, mean[D], var[D]] (f64, device) of an [n x obs_dim] observation batch."""
        n = obs.shape[0]
        out = out if out is not None else self.torch.empty(1 + 2 * self.obs_dim, dtype=self.torch.float64,
                                                           device=self.device)
        self._ck(lib().msk_gpu_obs_moments(self.h, _p(obs.contiguous()), int(n), _p(out), self._s(stream)))
        return out

    def obs_moments_fold(self, obs, acc, stream=None):
        """msk_gpu_obs_moments_fold: folds the batch moments of obs [n x obs_dim]
        into acc (f64 [1 + 2 obs_dim] {count, mean, var}, device, in place)."""
        self._ck(lib().msk_gpu_obs_moments_fold(self.h, _p(obs.contiguous()), int(obs.shape[0]), _p(acc),
                                                self._s(stream)))
        return acc

    def iteration_exchange(self, cap, obs, stats, norm, stats_out=None, nccl_comm=None, stream=None):
        """msk_gpu_iteration_exchange: drain + stats + obs moments, all-gather over
        nccl_comm (an ncclComm_t as int; None = single rank), rank-ordered merge on the
        device.  norm: f64 [1 + 2 obs_dim] device tensor {count, mean, var}, updated
        in place; returns stats_out (f64 [7])."""
        torch = self.torch
        stats_out = stats_out if stats_out is not None else torch.empty(7, dtype=torch.float64, device=self.device)
        self._ck(lib().msk_gpu_iteration_exchange(self.h, C.c_void_p(nccl_comm) if nccl_comm else None, int(cap),
                                                  _p(obs.contiguous()), _p(stats), _p(norm), _p(stats_out),
                                                  self._s(stream)))
        return stats_out

    def substeps(self, actions, n_substeps, stream=None):
        """msk_gpu_substeps: n (< 10) substeps of the continuous state, no env epilogue (parity diagnostics)."""
        a = actions if actions.dtype == self.torch.float32 and actions.is_contiguous() else actions.float().contiguous()
        self._ck(lib().msk_gpu_substeps(self.h, _p(a), int(n_substeps), None, None, self._s(stream)))

    def get_rng(self, stream=None):
        """(mt [E x 312] int64 (u64 bits), mti [E] int32): every env's mt19937_64 engine state."""
        torch = self.torch
        mt = self._empty(self.n, 312, dtype=torch.int64)
        mti = self._empty(self.n, dtype=torch.int32)
        self._ck(lib().msk_gpu_get_rng(self.h, _p(mt), _p(mti), self._s(stream)))
        return mt, mti

    def set_rng(self, mt, mti, stream=None):
        torch = self.torch
        a = torch.as_tensor(mt, device=self.device).view(torch.int64).contiguous() if mt is not None else None
        b = torch.as_tensor(mti, dtype=torch.int32, device=self.device).contiguous() if mti is not None else None
        self._ck(lib().msk_gpu_set_rng(self.h, _p(a), _p(b), self._s(stream)))
        self._keep = (a, b)

    def rng_serialize(self, env, stream=None):
        """Env e's engine state in the reference's Rng::serialize text (rng.hpp:56-61):
        the 312 state words, the word index, have_spare (0: Env draws no normals), spare."""
        mt, mti = self.get_rng(stream)
        self.torch.cuda.synchronize(self.device)
        words = mt[env].cpu().numpy().view("uint64")
        return " ".join(str(int(w)) for w in words) + f" {int(mti[env])} 0 0"

    def set_outcome_capacity(self, cap, stream=None):
        self._ck(lib().msk_gpu_set_outcome_capacity(self.h, int(cap), self._s(stream)))

    def outcomes_dropped(self):
        v = C.c_int64(0)
        self._ck(lib().msk_gpu_outcomes_dropped(self.h, C.byref(v)))
        return int(v.value)

    def rng_raw(self, env, n, stream=None):
        out = self._empty(n, dtype=self.torch.int64)  # raw u64 bits; view as uint64 on the host
        self._ck(lib().msk_gpu_rng_raw(self.h, int(env), int(n), _p(out), self._s(stream)))
        return out

    def fill_excitations(self, seed, step, actions=None, stream=None):
        actions = actions if actions is not None else self._empty(self.n, self.nm)
        self._ck(lib().msk_gpu_fill_excitations(self.h, C.c_uint64(seed), C.c_uint32(step), _p(actions),
                                                self._s(stream)))
        return actions
