"""TEST INFRASTRUCTURE ONLY — Python driver for the plain-C restatement
(oracle/msk_oracle.c) with the same batched verbs as oracle.ref.RefBatch.

Model JSON and clip CSV are read here with the reference's rules
(unknown keys rejected: /root/reference/proj/src/json_util.hpp:14-23,
model.cpp:94-196; clip columns: reference.cpp:35-86).
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

from .ref import EnvConfigC, _dp, _ip, _ptr, _up, env_config  # noqa: F401

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libmsk_oracle.so")


class ConfigError(ValueError):
    pass


def _check_keys(obj, allowed, where):
    if not isinstance(obj, dict):
        raise ConfigError(f"{where}: expected an object")
    for k in obj:
        if k not in allowed:
            raise ConfigError(f"{where}: unknown key '{k}'")


def load_model_json(path):
    """Flat arrays of a model (model.cpp:94-196 semantics)."""
    with open(path) as f:
        root = json.load(f)
    _check_keys(root, {"name", "root", "gravity", "joint_limit_stiffness", "links", "joints", "muscles",
                       "contacts", "contact_spheres", "key_bodies"}, path)
    if root["root"] not in ("fixed", "floating"):
        raise ConfigError("root must be 'fixed' or 'floating'")
    m = {"name": root["name"], "floating": root["root"] == "floating",
         "gravity": float(root.get("gravity", -9.81)),
         "joint_limit_stiffness": float(root.get("joint_limit_stiffness", 200.0))}
    links = root["links"]
    for l in links:
        _check_keys(l, {"name", "length", "mass", "inertia", "com"}, "links")
    m["link_length"] = np.array([l["length"] for l in links], dtype=np.float64)
    m["link_mass"] = np.array([l["mass"] for l in links], dtype=np.float64)
    m["link_inertia"] = np.array([l["inertia"] for l in links], dtype=np.float64)
    m["link_com"] = np.array([l["com"] for l in links], dtype=np.float64)
    joints = root.get("joints", [])
    for j in joints:
        _check_keys(j, {"name", "child", "parent", "anchor", "mount_angle", "limits", "damping"}, "joints")
    m["joint_parent"] = np.array([int(j["parent"]) for j in joints], dtype=np.int32)
    m["joint_child"] = np.array([int(j["child"]) for j in joints], dtype=np.int32)
    m["joint_anchor"] = np.array([j["anchor"] for j in joints], dtype=np.float64).reshape(-1, 2)
    m["joint_mount"] = np.array([j.get("mount_angle", 0.0) for j in joints], dtype=np.float64)
    m["joint_lo"] = np.array([j["limits"][0] if "limits" in j else -3.0 for j in joints], dtype=np.float64)
    m["joint_hi"] = np.array([j["limits"][1] if "limits" in j else 3.0 for j in joints], dtype=np.float64)
    m["joint_damping"] = np.array([j.get("damping", 0.0) for j in joints], dtype=np.float64)
    mus = root.get("muscles", [])
    for mu in mus:
        _check_keys(mu, {"name", "f_max", "l_opt", "v_max", "tau_act", "tau_deact", "tendon_slack", "via_points"},
                    "muscles")
    m["m_fmax"] = np.array([mu["f_max"] for mu in mus], dtype=np.float64)
    m["m_lopt"] = np.array([mu["l_opt"] for mu in mus], dtype=np.float64)
    m["m_vmax"] = np.array([mu.get("v_max", 10.0) for mu in mus], dtype=np.float64)
    m["m_tau_act"] = np.array([mu.get("tau_act", 0.010) for mu in mus], dtype=np.float64)
    m["m_tau_deact"] = np.array([mu.get("tau_deact", 0.040) for mu in mus], dtype=np.float64)
    m["m_slack"] = np.array([mu["tendon_slack"] for mu in mus], dtype=np.float64)
    starts = [0]
    vl, vo = [], []
    for mu in mus:
        for vp in mu["via_points"]:
            vl.append(int(vp[0]))
            vo.append([float(vp[1][0]), float(vp[1][1])])
        starts.append(len(vl))
    m["m_via_start"] = np.array(starts, dtype=np.int32)
    m["via_link"] = np.array(vl, dtype=np.int32)
    m["via_offset"] = np.array(vo, dtype=np.float64).reshape(-1, 2)
    cp = {"stiffness": 2.0e4, "damping": 500.0, "friction": 0.9, "smoothing_vel": 0.05}
    spheres = []
    if "contacts" in root:
        jc = root["contacts"]
        _check_keys(jc, {"stiffness", "damping", "friction", "smoothing_vel", "spheres"}, "contacts")
        for k in ("stiffness", "damping", "friction", "smoothing_vel"):
            cp[k] = float(jc.get(k, cp[k]))
        for s in jc.get("spheres", []):
            _check_keys(s, {"link", "offset", "radius"}, "contacts.spheres")
            spheres.append(s)
    # model.cpp:98 — top-level "contact_spheres" is accepted but ignored.
    m["contact"] = cp
    m["sphere_link"] = np.array([int(s["link"]) for s in spheres], dtype=np.int32)
    m["sphere_offset"] = np.array([s["offset"] for s in spheres], dtype=np.float64).reshape(-1, 2)
    m["sphere_radius"] = np.array([s["radius"] for s in spheres], dtype=np.float64)
    m["key_bodies"] = np.array([int(k) for k in root.get("key_bodies", [])], dtype=np.int32)
    m["n_links"], m["n_joints"], m["n_muscles"] = len(links), len(joints), len(mus)
    m["n_key"], m["n_spheres"] = len(m["key_bodies"]), len(spheres)
    m["nq"] = (3 if m["floating"] else 0) + len(joints)
    return m


def load_clip_csv(path, nq, nk):
    """Clip arrays in the reference layout (reference.cpp:35-86)."""
    with open(path) as f:
        header = f.readline().strip().split(",")
        data = np.loadtxt(f, delimiter=",", ndmin=2)
    c = 0

    def expect(name):
        nonlocal c
        if c >= len(header) or header[c] != name:
            raise ConfigError(f"expected column '{name}' at position {c}")
        c += 1
        return c - 1

    tcol = expect("time")
    rate = 50.0
    if data.shape[0] >= 2:
        dt = data[1, tcol] - data[0, tcol]
        if dt > 0:
            rate = 1.0 / dt
    q = np.stack([data[:, expect(f"q_{j}")] for j in range(nq)], axis=1)
    dq = np.stack([data[:, expect(f"dq_{j}")] for j in range(nq)], axis=1)
    kp = []
    for k in range(nk):
        kp.append(data[:, expect(f"key{k}_x")])
        kp.append(data[:, expect(f"key{k}_z")])
    key_pos = np.stack(kp, axis=1) if kp else np.zeros((data.shape[0], 0))
    ka = [data[:, expect(f"key{k}_angle")] for k in range(nk)]
    key_angle = np.stack(ka, axis=1) if ka else np.zeros((data.shape[0], 0))
    n_emg = 0
    while c + n_emg < len(header) and header[c + n_emg] == f"emg_{n_emg}":
        n_emg += 1
    emg = data[:, c:c + n_emg].copy()
    c += n_emg
    return dict(rate=rate, q=np.ascontiguousarray(q), dq=np.ascontiguousarray(dq),
                key_pos=np.ascontiguousarray(key_pos), key_angle=np.ascontiguousarray(key_angle),
                emg=np.ascontiguousarray(emg), frames=data.shape[0])


class OmModel(C.Structure):
    _fields_ = [
        ("floating", C.c_int32), ("n_links", C.c_int32), ("n_joints", C.c_int32), ("n_muscles", C.c_int32),
        ("n_key", C.c_int32), ("n_spheres", C.c_int32), ("gravity", C.c_double),
        ("joint_limit_stiffness", C.c_double),
        ("link_length", _dp), ("link_mass", _dp), ("link_inertia", _dp), ("link_com", _dp),
        ("joint_parent", _ip), ("joint_anchor", _dp), ("joint_mount", _dp), ("joint_lo", _dp),
        ("joint_hi", _dp), ("joint_damping", _dp),
        ("m_fmax", _dp), ("m_lopt", _dp), ("m_vmax", _dp), ("m_tau_act", _dp), ("m_tau_deact", _dp),
        ("m_slack", _dp), ("m_via_start", _ip), ("via_link", _ip), ("via_offset", _dp),
        ("sphere_link", _ip), ("sphere_offset", _dp), ("sphere_radius", _dp),
        ("contact_k", C.c_double), ("contact_c", C.c_double), ("contact_mu", C.c_double),
        ("contact_vs", C.c_double), ("key_bodies", _ip),
    ]


class OmClip(C.Structure):
    _fields_ = [("frames", C.c_int32), ("q", _dp), ("dq", _dp), ("key_pos", _dp), ("key_angle", _dp),
                ("n_emg", C.c_int32), ("emg", _dp)]


class OmRewardConfig(C.Structure):
    _fields_ = [("mode", C.c_int32), ("n_emg_channels", C.c_int32), ("w_emg", C.c_double),
                ("w_power", C.c_double), ("emg_channel_map", _ip)]


class OmEnv(C.Structure):
    _fields_ = [
        ("q", _dp), ("dq", _dp), ("act", _dp), ("l_m", _dp), ("v_m", _dp), ("f_m", _dp), ("t", C.c_double),
        ("t_index", C.c_int32), ("start_index", C.c_int32), ("steps", C.c_int32), ("done", C.c_int32),
        ("eval_mode", C.c_int32), ("mt", C.c_uint64 * 312), ("mti", C.c_int32), ("failure_ema", _dp),
        ("n_outcomes", C.c_int32), ("outcome_cap", C.c_int32), ("outcome_bin", _ip), ("outcome_failed", _up),
    ]


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(ORACLE_SO):
            raise FileNotFoundError(f"{ORACLE_SO} missing — run `make -C oracle`")
        L = C.CDLL(ORACLE_SO)
        P = C.POINTER
        L.om_force_length_active.restype = C.c_double
        L.om_force_length_active.argtypes = [C.c_double]
        L.om_force_velocity.restype = C.c_double
        L.om_force_velocity.argtypes = [C.c_double]
        L.om_force_passive.restype = C.c_double
        L.om_force_passive.argtypes = [C.c_double]
        L.om_mtu_force.restype = C.c_double
        L.om_mtu_force.argtypes = [C.c_double] * 4
        L.om_activation_step.restype = C.c_double
        L.om_activation_step.argtypes = [C.c_double] * 5
        L.om_wrap_angle.restype = C.c_double
        L.om_wrap_angle.argtypes = [C.c_double]
        L.om_mass_matrix.argtypes = [P(OmModel), _dp, _dp]
        L.om_moment_arms.argtypes = [P(OmModel), _dp, _dp]
        L.om_bias_forces.argtypes = [P(OmModel), _dp, _dp, _dp]
        L.om_contact_forces.argtypes = [P(OmModel), _dp, _dp, _dp, _dp]
        L.om_mtu_length.restype = C.c_double
        L.om_mtu_length.argtypes = [P(OmModel), _dp, C.c_int32]
        L.om_mechanical_energy.restype = C.c_double
        L.om_mechanical_energy.argtypes = [P(OmModel), _dp, _dp]
        L.om_key_body_state.argtypes = [P(OmModel), _dp, _dp, _dp]
        L.om_make_initial_state.argtypes = [P(OmModel), _dp, _dp, C.c_double, _dp, _dp, _dp, _dp, _dp, _dp]
        L.om_step.restype = C.c_int32
        L.om_step.argtypes = [P(OmModel), _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp]
        L.om_substep.restype = C.c_int32
        L.om_substep.argtypes = [P(OmModel), _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp]
        L.om_rng_seed.argtypes = [P(OmEnv), C.c_uint64]
        L.om_rng_raw.restype = C.c_uint64
        L.om_rng_raw.argtypes = [P(OmEnv)]
        L.om_env_init.argtypes = [P(OmModel), P(OmClip), P(EnvConfigC), P(OmEnv), C.c_uint64]
        L.om_env_reset.restype = C.c_int32
        L.om_env_reset.argtypes = [P(OmModel), P(OmClip), P(EnvConfigC), P(OmEnv), _dp]
        L.om_env_reset_to_frame.restype = C.c_int32
        L.om_env_reset_to_frame.argtypes = [P(OmModel), P(OmClip), P(EnvConfigC), P(OmEnv), C.c_int32, _dp]
        L.om_env_observe.argtypes = [P(OmModel), P(OmClip), P(OmEnv), _dp]
        L.om_env_tracking_error.argtypes = [P(OmModel), P(OmClip), P(OmEnv), _dp]
        L.om_env_step.restype = C.c_int32
        L.om_env_step.argtypes = [P(OmModel), P(OmClip), P(EnvConfigC), P(OmRewardConfig), P(OmEnv), _dp, _dp,
                                  _dp, _dp, _dp, _dp]
        L.om_sampler_record.argtypes = [P(EnvConfigC), P(OmEnv), C.c_int32, C.c_int32]
        L.om_excitation.restype = C.c_double
        L.om_excitation.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_int32]
        L.om_obs_dim.restype = C.c_int32
        L.om_obs_dim.argtypes = [P(OmModel)]
        L.om_mlp_param_count.restype = C.c_int64
        L.om_mlp_param_count.argtypes = [C.c_int32, C.c_int32, C.c_int32]
        L.om_mlp_init.argtypes = [_dp, C.c_int32, C.c_int32, C.c_int32, C.c_uint64, C.c_double]
        L.om_mlp_forward_sigmoid.argtypes = [_dp, C.c_int32, C.c_int32, _dp, C.c_int32, _dp]
        L.om_disc_reward.restype = C.c_double
        L.om_disc_reward.argtypes = [C.c_double]
        L.om_delta_dim.restype = C.c_int32
        L.om_delta_dim.argtypes = [P(OmModel)]
        _LIB = L
    return _LIB


class OracleModel:
    """Keeps the numpy arrays alive behind an OmModel struct."""

    def __init__(self, path):
        self.d = load_model_json(path)
        d = self.d
        self._keep = []

        def dp(a):
            a = np.ascontiguousarray(a, dtype=np.float64).ravel()
            self._keep.append(a)
            return a.ctypes.data_as(_dp) if a.size else None

        def ip(a):
            a = np.ascontiguousarray(a, dtype=np.int32).ravel()
            self._keep.append(a)
            return a.ctypes.data_as(_ip) if a.size else None

        cp = d["contact"]
        self.s = OmModel(
            int(d["floating"]), d["n_links"], d["n_joints"], d["n_muscles"], d["n_key"], d["n_spheres"],
            d["gravity"], d["joint_limit_stiffness"],
            dp(d["link_length"]), dp(d["link_mass"]), dp(d["link_inertia"]), dp(d["link_com"]),
            ip(d["joint_parent"]), dp(d["joint_anchor"]), dp(d["joint_mount"]), dp(d["joint_lo"]),
            dp(d["joint_hi"]), dp(d["joint_damping"]),
            dp(d["m_fmax"]), dp(d["m_lopt"]), dp(d["m_vmax"]), dp(d["m_tau_act"]), dp(d["m_tau_deact"]),
            dp(d["m_slack"]), ip(d["m_via_start"]), ip(d["via_link"]), dp(d["via_offset"]),
            ip(d["sphere_link"]), dp(d["sphere_offset"]), dp(d["sphere_radius"]),
            cp["stiffness"], cp["damping"], cp["friction"], cp["smoothing_vel"], ip(d["key_bodies"]))
        self.nq, self.nm, self.nk = d["nq"], d["n_muscles"], d["n_key"]
        self.n_links = d["n_links"]
        self.floating = d["floating"]
        self.ref = C.byref(self.s)

    # model-level functions
    def mass_matrix(self, q):
        q = np.ascontiguousarray(q, dtype=np.float64)
        M = np.zeros((self.nq, self.nq))
        lib().om_mass_matrix(self.ref, _ptr(q, _dp), _ptr(M, _dp))
        return M

    def moment_arms(self, q):
        q = np.ascontiguousarray(q, dtype=np.float64)
        J = np.zeros((self.nm, self.nq))
        lib().om_moment_arms(self.ref, _ptr(q, _dp), _ptr(J, _dp))
        return J

    def bias_forces(self, q, dq):
        q = np.ascontiguousarray(q, dtype=np.float64)
        dq = np.ascontiguousarray(dq, dtype=np.float64)
        c = np.zeros(self.nq)
        lib().om_bias_forces(self.ref, _ptr(q, _dp), _ptr(dq, _dp), _ptr(c, _dp))
        return c

    def contact_forces(self, q, dq):
        q = np.ascontiguousarray(q, dtype=np.float64)
        dq = np.ascontiguousarray(dq, dtype=np.float64)
        tau = np.zeros(self.nq)
        sf = np.zeros((max(1, self.d["n_spheres"]), 2))
        lib().om_contact_forces(self.ref, _ptr(q, _dp), _ptr(dq, _dp), _ptr(tau, _dp), _ptr(sf, _dp))
        return tau, sf[: self.d["n_spheres"]]

    def mtu_length(self, q, m):
        q = np.ascontiguousarray(q, dtype=np.float64)
        return lib().om_mtu_length(self.ref, _ptr(q, _dp), m)

    def mechanical_energy(self, q, dq):
        q = np.ascontiguousarray(q, dtype=np.float64)
        dq = np.ascontiguousarray(dq, dtype=np.float64)
        return lib().om_mechanical_energy(self.ref, _ptr(q, _dp), _ptr(dq, _dp))

    def key_bodies(self, q):
        q = np.ascontiguousarray(q, dtype=np.float64)
        pos = np.zeros((max(1, self.nk), 2))
        ang = np.zeros(max(1, self.nk))
        lib().om_key_body_state(self.ref, _ptr(q, _dp), _ptr(pos, _dp), _ptr(ang, _dp))
        return pos[: self.nk], ang[: self.nk]

    def substep(self, q, dq, act, l_m, v_m, f_m, u):
        """One 2 ms substep in place on float64 copies; returns (state dict, qdd, diverged)."""
        s = {k: np.array(v, dtype=np.float64) for k, v in dict(q=q, dq=dq, act=act, l_m=l_m, v_m=v_m,
                                                               f_m=f_m).items()}
        u = np.ascontiguousarray(u, dtype=np.float64)
        qdd = np.zeros(self.nq)
        bad = lib().om_substep(self.ref, *[_ptr(s[k], _dp) for k in ("q", "dq", "act", "l_m", "v_m", "f_m")],
                               _ptr(u, _dp), _ptr(qdd, _dp))
        return s, qdd, bool(bad)


class OracleBatch:
    """E oracle environments with the RefBatch verbs."""

    def __init__(self, model_path, clip_path, n_envs, base_seed=0x5EED, cfg=None, reward_mode=0, w_emg=100.0,
                 w_power=0.05, emg_map=(), global_env_offset=0, outcome_cap=64):
        self.model = OracleModel(model_path)
        md = self.model.d
        self.nq, self.nm, self.nk, self.n_links = md["nq"], md["n_muscles"], md["n_key"], md["n_links"]
        self.nj = md["n_joints"]
        self.floating = md["floating"]
        self.cfg = cfg if cfg is not None else env_config()
        self.bins = max(1, int(self.cfg.adaptive_bins))
        self.clip = load_clip_csv(clip_path, self.nq, self.nk)
        cl = self.clip
        self.frames = cl["frames"]
        self.cs = OmClip(cl["frames"], _ptr(cl["q"], _dp), _ptr(cl["dq"], _dp),
                         _ptr(cl["key_pos"], _dp) if cl["key_pos"].size else None,
                         _ptr(cl["key_angle"], _dp) if cl["key_angle"].size else None, cl["emg"].shape[1],
                         _ptr(cl["emg"], _dp) if cl["emg"].size else None)
        self._emg = np.asarray(emg_map, dtype=np.int32)
        self.rc = OmRewardConfig(int(reward_mode), len(self._emg), float(w_emg), float(w_power),
                                 _ptr(self._emg, _ip) if len(self._emg) else None)
        L = lib()
        self.obs_dim = L.om_obs_dim(self.model.ref)
        self.delta_dim = L.om_delta_dim(self.model.ref)
        self.n = n_envs
        nq, nm = self.nq, self.nm
        self.arr = dict(q=np.zeros((n_envs, nq)), dq=np.zeros((n_envs, nq)), act=np.zeros((n_envs, nm)),
                        l_m=np.zeros((n_envs, nm)), v_m=np.zeros((n_envs, nm)), f_m=np.zeros((n_envs, nm)),
                        ema=np.zeros((n_envs, self.bins)), ob=np.zeros((n_envs, outcome_cap), dtype=np.int32),
                        of=np.zeros((n_envs, outcome_cap), dtype=np.uint8))
        self.envs = []
        for e in range(n_envs):
            a = self.arr
            env = OmEnv()
            env.q, env.dq = _ptr(a["q"][e], _dp), _ptr(a["dq"][e], _dp)
            env.act, env.l_m = _ptr(a["act"][e], _dp), _ptr(a["l_m"][e], _dp)
            env.v_m, env.f_m = _ptr(a["v_m"][e], _dp), _ptr(a["f_m"][e], _dp)
            env.failure_ema = _ptr(a["ema"][e], _dp)
            env.outcome_cap = outcome_cap
            env.outcome_bin = _ptr(a["ob"][e], _ip)
            env.outcome_failed = _ptr(a["of"][e], _up)
            L.om_env_init(self.model.ref, C.byref(self.cs), C.byref(self.cfg), C.byref(env),
                          C.c_uint64(base_seed + global_env_offset + e))
            self.envs.append(env)

    def set_eval_mode(self, ev=True):
        for env in self.envs:
            env.eval_mode = int(bool(ev))

    def reset(self, mask=None):
        obs = np.zeros((self.n, self.obs_dim))
        frames = np.full(self.n, -1, dtype=np.int32)
        L = lib()
        for e, env in enumerate(self.envs):
            if mask is not None and not mask[e]:
                continue
            L.om_env_reset(self.model.ref, C.byref(self.cs), C.byref(self.cfg), C.byref(env), _ptr(obs[e], _dp))
            frames[e] = env.start_index
        return obs, frames

    def reset_to_frame(self, frames, mask=None):
        fr = np.broadcast_to(np.asarray(frames, dtype=np.int32), (self.n,))
        obs = np.zeros((self.n, self.obs_dim))
        L = lib()
        for e, env in enumerate(self.envs):
            if mask is not None and not mask[e]:
                continue
            if L.om_env_reset_to_frame(self.model.ref, C.byref(self.cs), C.byref(self.cfg), C.byref(env),
                                       int(fr[e]), _ptr(obs[e], _dp)):
                raise ValueError("reset_to_frame: frame out of range")
        return obs

    def step(self, actions):
        a = np.ascontiguousarray(actions, dtype=np.float64).reshape(self.n, self.nm)
        obs = np.zeros((self.n, self.obs_dim))
        delta = np.zeros((self.n, self.delta_dim))
        raux = np.zeros(self.n)
        flags = np.zeros(self.n, dtype=np.uint8)
        power = np.zeros((self.n, self.nm))
        grf = np.zeros((self.n, self.n_links, 2))
        L = lib()
        for e, env in enumerate(self.envs):
            flags[e] = L.om_env_step(self.model.ref, C.byref(self.cs), C.byref(self.cfg), C.byref(self.rc),
                                     C.byref(env), _ptr(a[e], _dp), _ptr(obs[e], _dp), _ptr(delta[e], _dp),
                                     _ptr(raux[e:e + 1], _dp), _ptr(power[e], _dp), _ptr(grf[e], _dp))
        return dict(obs=obs, delta=delta, reward_aux=raux, flags=flags, power=power, grf=grf)

    def observe(self):
        obs = np.zeros((self.n, self.obs_dim))
        for e, env in enumerate(self.envs):
            lib().om_env_observe(self.model.ref, C.byref(self.cs), C.byref(env), _ptr(obs[e], _dp))
        return obs

    def tracking_error(self):
        d = np.zeros((self.n, self.delta_dim))
        for e, env in enumerate(self.envs):
            lib().om_env_tracking_error(self.model.ref, C.byref(self.cs), C.byref(env), _ptr(d[e], _dp))
        return d

    def get_state(self):
        a = self.arr
        ints = np.array([[env.t_index, env.start_index, env.steps, env.done] for env in self.envs],
                        dtype=np.int32).reshape(self.n, 4)
        return dict(q=a["q"].copy(), dq=a["dq"].copy(), act=a["act"].copy(), l_m=a["l_m"].copy(),
                    v_m=a["v_m"].copy(), f_m=a["f_m"].copy(), t=np.array([env.t for env in self.envs]), ints=ints)

    def set_state(self, s):
        for k in ("q", "dq", "act", "l_m", "v_m", "f_m"):
            self.arr[k][...] = s[k]
        for e, env in enumerate(self.envs):
            env.t = float(s["t"][e])
            env.t_index, env.start_index, env.steps, env.done = [int(x) for x in s["ints"][e]]

    def get_sampler(self):
        return self.arr["ema"].copy()

    def set_sampler(self, ema):
        self.arr["ema"][...] = np.broadcast_to(ema, self.arr["ema"].shape)

    def drain_outcomes(self, cap=64):
        bins = np.zeros((self.n, cap), dtype=np.int32)
        failed = np.zeros((self.n, cap), dtype=np.uint8)
        counts = np.zeros(self.n, dtype=np.int32)
        for e, env in enumerate(self.envs):
            n = min(env.n_outcomes, cap, env.outcome_cap)
            counts[e] = env.n_outcomes
            bins[e, :n] = self.arr["ob"][e, :n]
            failed[e, :n] = self.arr["of"][e, :n]
            env.n_outcomes = 0
        return bins, failed, counts

    def record_own_outcomes(self):
        for e, env in enumerate(self.envs):
            n = min(env.n_outcomes, env.outcome_cap)
            for i in range(n):
                lib().om_sampler_record(C.byref(self.cfg), C.byref(env), int(self.arr["ob"][e, i]),
                                        int(self.arr["of"][e, i]))
            env.n_outcomes = 0

    def rng_raw(self, env, n):
        return np.array([lib().om_rng_raw(C.byref(self.envs[env])) for _ in range(n)], dtype=np.uint64)

    def get_rng(self):
        """(mt [E x 312] uint64, mti [E] int32) of every env (rng.hpp:71 engine state)."""
        mt = np.array([np.ctypeslib.as_array(env.mt) for env in self.envs], dtype=np.uint64)
        return mt, np.array([env.mti for env in self.envs], dtype=np.int32)

    def set_rng(self, mt, mti):
        for e, env in enumerate(self.envs):
            for i in range(312):
                env.mt[i] = int(mt[e, i])
            env.mti = int(mti[e])

    def rng_serialize(self, env):
        """Rng::serialize() text (rng.hpp:56-61): 312 words, index, have_spare 0, spare 0."""
        mt, mti = self.get_rng()
        return " ".join(str(int(w)) for w in mt[env]) + f" {int(mti[env])} 0 0"


def excitations(seed, step, n_envs, nm, global_env_offset=0):
    L = lib()
    out = np.zeros((n_envs, nm))
    for e in range(n_envs):
        for m in range(nm):
            out[e, m] = L.om_excitation(C.c_uint64(seed), step, global_env_offset + e, m)
    return out


# ---- discriminator (nn.cpp Mlp with Head::Sigmoid) --------
def mlp_param_count(n_in, hidden, n_out=1):
    return int(lib().om_mlp_param_count(n_in, hidden, n_out))


def mlp_init(n_in, hidden, seed, n_out=1, final_init_scale=1.0):
    """Mlp(MlpShape{in, hidden, out}, seed) parameters (nn.cpp:16-38), f64 flat."""
    theta = np.zeros(mlp_param_count(n_in, hidden, n_out))
    lib().om_mlp_init(_ptr(theta, _dp), n_in, hidden, n_out, C.c_uint64(seed), float(final_init_scale))
    return theta


def mlp_forward_sigmoid(theta, n_in, hidden, x):
    """D(x) per row (nn.cpp:54-73, Sigmoid head, out = 1)."""
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, n_in)
    y = np.zeros(x.shape[0])
    theta = np.ascontiguousarray(theta, dtype=np.float64)
    lib().om_mlp_forward_sigmoid(_ptr(theta, _dp), n_in, hidden, _ptr(x, _dp), x.shape[0], _ptr(y, _dp))
    return y


def disc_reward(theta, n_in, hidden, delta):
    """reward_from_discriminator: -log(1 - clamp(D(delta), 1e-4, 1 - 1e-4))."""
    L = lib()
    return np.array([L.om_disc_reward(d) for d in mlp_forward_sigmoid(theta, n_in, hidden, delta)])
