"""CPU tests of the product library's boundary (no GPU compute).

* libmsk_b200.so loads and exports every entry point include/msk_gpu.h declares;
* the host model/clip ingest accepts and rejects exactly what the
  reference's parse_model_json / ModelSpec::validate / load_reference do;
* without a B200 the context refuses to start (no CPU fallback).
"""
import ctypes as C
import json
import os
import re

import pytest

from conftest import ROOT, model_paths

HEADER = os.path.join(ROOT, "include", "msk_gpu.h")


def _lib():
    import paper_2603_29332_b200 as pk

    return pk.lib()


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(msk_gpu_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = _lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s


def test_library_is_sm100a_only():
    so = os.path.join(ROOT, "paper_2603_29332_b200", "libmsk_b200.so")
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out), out


def _validate(model, clip=None):
    import paper_2603_29332_b200 as pk

    L = _lib()
    L.msk_gpu_validate.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(pk._Dims)]
    L.msk_gpu_validate.restype = C.c_int
    d = pk._Dims()
    rc = L.msk_gpu_validate(model.encode(), clip.encode() if clip else None, C.byref(d))
    return rc, d, L.msk_gpu_last_error(None).decode()


@pytest.mark.parametrize("name", ["pendulum1_m2", "arm2_m6", "walker5_m16", "wb700", "wb700_fixed"])
def test_validate_bundled_models(assets, name):
    mp, cp = model_paths(name)
    rc, d, err = _validate(mp, cp)
    assert rc == 0, err
    js = json.load(open(mp))
    nq = (3 if js["root"] == "floating" else 0) + len(js["joints"])
    assert d.nq == nq and d.n_muscles == len(js["muscles"])
    assert d.obs_dim == 3 * nq + 6 * len(js["key_bodies"]) + 4 * len(js["muscles"])  # env.cpp:165-168
    assert d.delta_dim == 3 + len(js["joints"]) + 2 * len(js["key_bodies"])  # env.hpp:25-27
    assert d.frames == 1101


def _mutated(tmp_path, name, fn):
    mp, _ = model_paths(name)
    js = json.load(open(mp))
    fn(js)
    p = tmp_path / "m.json"
    p.write_text(json.dumps(js))
    return str(p)


@pytest.mark.parametrize("mut,msg", [
    (lambda js: js.update(bogus=1), "unknown key 'bogus'"),
    (lambda js: js["links"][0].update(mass=-1.0), "mass must be > 0"),
    (lambda js: js["muscles"][0]["via_points"].pop(), "at least 2 via points"),
    (lambda js: js["muscles"][0].update(tau_act=0.5), "tau_act <= tau_deact"),
    (lambda js: js["joints"][1].update(parent=5), "parent"),
    (lambda js: js.update(root="hinged"), "root must be 'fixed' or 'floating'"),
    (lambda js: js["joints"][0].update(extra=0), "unknown key 'extra'"),
])
def test_validate_rejects_like_reference(assets, tmp_path, mut, msg):
    p = _mutated(tmp_path, "arm2_m6", mut)
    rc, _, err = _validate(p)
    assert rc == 1 and msg in err, err


def test_contact_spheres_top_level_key_accepted_but_ignored(assets, tmp_path):
    # model.cpp:98 accepts "contact_spheres" and reads spheres only from contacts.spheres
    p = _mutated(tmp_path, "arm2_m6", lambda js: js.update(contact_spheres=[{"link": 0}]))
    rc, d, err = _validate(p)
    assert rc == 0 and d.n_spheres == 0, err


def test_clip_validation(assets, tmp_path):
    mp, cp = model_paths("arm2_m6")
    lines = open(cp).read().splitlines()
    bad = tmp_path / "bad.csv"
    bad.write_text("\n".join([lines[0].replace("dq_0", "dq_x")] + lines[1:]) + "\n")
    rc, _, err = _validate(mp, str(bad))
    assert rc == 1 and "expected column 'dq_0'" in err
    slow = tmp_path / "slow.csv"  # 25 Hz clip
    rows = [lines[0]] + [",".join([str(float(r.split(",")[0]) * 2)] + r.split(",")[1:]) for r in lines[1:]]
    slow.write_text("\n".join(rows) + "\n")
    rc, _, err = _validate(mp, str(slow))
    assert rc == 1 and "50 Hz" in err


def test_no_cpu_fallback_without_gpu(assets):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2603_29332_b200 as pk

    mp, cp = model_paths("arm2_m6")
    with pytest.raises(pk.MskError) as ei:
        pk.EnvBatch(mp, cp, 4, device=0)
    assert ei.value.code == 3


def test_host_mlp_init_matches_oracle_and_reference_rng():
    """msk_mlp_init (host C++, product side) == the oracle's Mlp init, which the
    golden fixture pins to the reference's Rng stream (nn.cpp:16-38)."""
    import numpy as np

    import paper_2603_29332_b200 as pk
    from oracle.oracle import mlp_init

    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "mlp_seed7.npz"))
    assert np.array_equal(pk.mlp_init(9, 16, 7), g["small"])
    big = pk.mlp_init(102, 256, 7)
    assert np.array_equal(big, mlp_init(102, 256, 7))
    assert np.array_equal(big[:512], g["big_head"]) and np.sum(big) == g["big_sum"][0]
    assert np.array_equal(pk.mlp_init(5, 32, 1, final_init_scale=0.0)[-33:], np.zeros(33))


def test_new_entry_points_fail_cleanly_without_gpu_or_bad_args():
    """Policy / rollout / discriminator entry points report errors (no crash) on
    bad shapes, and on a host without a GPU report a CUDA error instead of
    falling back to the CPU."""
    import numpy as np

    import paper_2603_29332_b200 as pk

    L = pk.lib()
    assert L.msk_mlp_param_count(0, 16, 1) < 0
    th = np.zeros(4)
    assert L.msk_mlp_init(th.ctypes.data, 0, 16, 1, 7, 1.0) != 0
    h = C.c_void_p()
    # hidden width not a multiple of 64 -> contract error (status 1) before any device work
    pi = np.zeros(10)
    rc = L.msk_policy_create(8, 4, 48, pi.ctypes.data, pi.size, 1.0, 0.0, pi.ctypes.data, pi.ctypes.data, pi.size,
                             20, 0.05, 16, 0, C.byref(h))
    assert rc == 1 and not h.value
    assert b"multiple of 64" in L.msk_policy_last_error(None)
    # wrong parameter count -> contract error
    rc = L.msk_policy_create(8, 4, 64, pi.ctypes.data, pi.size, 1.0, 0.0, pi.ctypes.data, pi.ctypes.data, pi.size,
                             20, 0.05, 16, 0, C.byref(h))
    assert rc == 1 and b"parameter count" in L.msk_policy_last_error(None)
    r = C.c_void_p()
    assert L.msk_rollout_create(0, 8, 1, 1, 1, 0, C.byref(r)) != 0 and not r.value


def test_minibatch_oracle_is_a_bijection():
    """The oracle's Feistel shuffle (rollout.cu msk_rollout_minibatch) permutes
    [0, n) for ragged n, and depends on (seed, epoch)."""
    import numpy as np

    from oracle.policy import feistel_permutation, minibatch_key

    for n in (1, 2, 3, 7, 296, 1000, 4097):
        p = feistel_permutation(n, minibatch_key(5, 0))
        assert np.array_equal(np.sort(p), np.arange(n))
    assert not np.array_equal(feistel_permutation(500, minibatch_key(5, 0)), feistel_permutation(500, minibatch_key(5, 1)))


def test_exchange_and_minibatch_entry_points_fail_cleanly():
    """msk_gpu_iteration_exchange / msk_rollout_minibatch report contract errors
    (status 1) on null contexts and bad arguments — no crash, no CPU fallback."""
    import paper_2603_29332_b200 as pk

    L = pk.lib()
    assert L.msk_gpu_iteration_exchange(None, None, 8, None, None, None, None, None) == 1
    assert L.msk_rollout_minibatch(None, 1, 0, 0, 8, *([None] * 8), None) == 1
    assert b"null" in L.msk_rollout_last_error(None)
