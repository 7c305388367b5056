"""Multi-process (gloo, world_size 2, CPU) tests of the iteration exchange.

The GPU path uses the same pack/all_gather/merge code with NCCL and the
device merge kernel; here the outcome merge runs on the host
(merge_outcomes_host), which the GPU test compares bit-exactly with
msk_gpu_merge_outcomes.
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_29332_b200 import dist as mdist

N_ENVS, CAP, OBS_DIM, BINS, DECAY = 6, 5, 7, 10, 0.99


def rank_data(rank):
    g = np.random.default_rng(100 + rank)
    counts = g.integers(0, CAP + 2, N_ENVS)  # some envs overflow the cap
    bins = g.integers(0, BINS, (N_ENVS, CAP))
    failed = g.integers(0, 2, (N_ENVS, CAP))
    stats = g.normal(size=mdist.N_STATS)
    obs = g.normal(size=(N_ENVS, OBS_DIM)) * (1 + rank)
    return (torch.tensor(bins, dtype=torch.int32), torch.tensor(failed, dtype=torch.int32),
            torch.tensor(counts, dtype=torch.int32), torch.tensor(stats), torch.tensor(obs))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    bins, failed, counts, stats, obs = rank_data(rank)
    block = mdist.pack_block(bins, failed, counts, stats, mdist.batch_moments(obs), OBS_DIM)
    blocks = mdist.exchange(block)
    ema0 = np.linspace(0, 0.2, BINS)
    st, norm, ema = mdist.merged_iteration(blocks, N_ENVS, CAP, OBS_DIM, (0.0, np.zeros(OBS_DIM), np.ones(OBS_DIM)),
                                           ema0, DECAY)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), stats=st.numpy(), count=norm[0], mean=norm[1], var=norm[2],
             ema=ema)
    dist.destroy_process_group()


def test_pack_roundtrip():
    bins, failed, counts, stats, obs = rank_data(0)
    norm = mdist.batch_moments(obs)
    p = mdist.unpack_block(mdist.pack_block(bins, failed, counts, stats, norm, OBS_DIM), N_ENVS, CAP, OBS_DIM)
    assert torch.equal(p["bins"], bins) and torch.equal(p["failed"], failed) and torch.equal(p["counts"], counts)
    assert torch.equal(p["stats"], stats) and torch.equal(p["norm"], norm)


def test_two_rank_exchange_matches_single_rank_ordered_merge(tmp_path):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    r0, r1 = (np.load(tmp_path / f"r{r}.npz") for r in range(2))
    for k in r0.files:  # every rank ends bit-identical
        assert np.array_equal(r0[k], r1[k]), k
    # single-rank reference: concatenation in global env order, merged in order
    d0, d1 = rank_data(0), rank_data(1)
    bins = torch.cat([d0[0], d1[0]])
    failed = torch.cat([d0[1], d1[1]])
    counts = torch.cat([d0[2], d1[2]])
    ema = mdist.merge_outcomes_host(np.linspace(0, 0.2, BINS), bins, failed, counts, DECAY)
    assert np.array_equal(ema, r0["ema"])
    assert np.array_equal(r0["stats"], (d0[3] + d1[3]).numpy()) or np.allclose(r0["stats"], (d0[3] + d1[3]).numpy(),
                                                                              rtol=0, atol=0)
    # RunningNorm parallel fold == one update with all rows (up to rounding)
    allobs = np.concatenate([d0[4].numpy(), d1[4].numpy()])
    assert abs(r0["count"] - 2 * N_ENVS) == 0
    assert np.allclose(r0["mean"], allobs.mean(0), rtol=1e-12, atol=1e-12)
    assert np.allclose(r0["var"], allobs.var(0), rtol=1e-12, atol=1e-12)


def test_host_merge_equals_oracle_sampler_record(assets):
    """merge_outcomes_host follows AdaptiveSampler::record exactly (oracle, env.cpp:34-37)."""
    from conftest import model_paths
    from oracle.oracle import OracleBatch, lib
    from oracle.ref import env_config

    mp_, cp = model_paths("arm2_m6")
    cfg = env_config(adaptive_bins=BINS, adaptive_decay=DECAY)
    o = OracleBatch(mp_, cp, 1, cfg=cfg)
    o.set_sampler(np.linspace(0, 0.2, BINS))
    d = rank_data(0)
    for g in range(N_ENVS):
        for i in range(min(int(d[2][g]), CAP)):
            lib().om_sampler_record(C.byref(cfg), C.byref(o.envs[0]), int(d[0][g, i]), int(d[1][g, i]))
    host = mdist.merge_outcomes_host(np.linspace(0, 0.2, BINS), d[0], d[1], d[2], DECAY)
    assert np.array_equal(o.get_sampler()[0], host)


@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a GPU")
@pytest.mark.gpu
def test_device_merge_bit_exact_with_host(assets):
    import paper_2603_29332_b200 as pk
    from conftest import model_paths

    mp_, cp = model_paths("arm2_m6")
    g = pk.EnvBatch(mp_, cp, 3, cfg=pk.EnvConfig(adaptive_bins=BINS, adaptive_decay=DECAY))
    ema0 = np.linspace(0, 0.2, BINS)
    g.set_sampler(torch.as_tensor(ema0, device=g.device))
    d0, d1 = rank_data(0), rank_data(1)
    bins = torch.cat([d0[0], d1[0]]).cuda()
    failed = torch.cat([d0[1], d1[1]]).to(torch.uint8).cuda()
    counts = torch.cat([d0[2], d1[2]]).cuda()
    g.merge_outcomes(bins, failed, counts)
    host = mdist.merge_outcomes_host(ema0, bins.cpu(), failed.cpu(), counts.cpu(), DECAY)
    got = g.get_sampler().cpu().numpy()
    for e in range(3):
        assert np.array_equal(got[e], host)
    g.close()


@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a GPU")
@pytest.mark.gpu
def test_device_merge_large_bit_exact_with_host(assets):
    """Chunked block-scan merge: > 1024 envs and > 4096 outcomes in one chunk."""
    import paper_2603_29332_b200 as pk
    from conftest import model_paths

    mp_, cp = model_paths("arm2_m6")
    g = pk.EnvBatch(mp_, cp, 2, cfg=pk.EnvConfig(adaptive_bins=BINS, adaptive_decay=DECAY))
    ema0 = np.linspace(0.05, 0.3, BINS)
    g.set_sampler(torch.as_tensor(ema0, device=g.device))
    rng = np.random.default_rng(9)
    n, cap = 5000, 8
    counts = torch.as_tensor(rng.integers(0, cap + 3, n), dtype=torch.int32)  # some exceed cap (clamped)
    bins = torch.as_tensor(rng.integers(0, BINS, (n, cap)), dtype=torch.int32)
    failed = torch.as_tensor(rng.integers(0, 2, (n, cap)), dtype=torch.uint8)
    g.merge_outcomes(bins.cuda(), failed.cuda(), counts.cuda())
    host = mdist.merge_outcomes_host(ema0, bins, failed, counts, DECAY)
    got = g.get_sampler().cpu().numpy()
    assert np.array_equal(got[0], host) and np.array_equal(got[1], host)
    g.close()


def test_device_norm_fold_matches_host_fold():
    """The on-device RunningNorm fold (no host sync) == the numpy fold, bit for bit,
    including the first-batch branch (nn.cpp:257-262) and empty batches."""
    import numpy as np
    import torch

    from paper_2603_29332_b200 import dist as mdist

    rng = np.random.default_rng(5)
    d = 7
    host = (0.0, np.zeros(d), np.ones(d))
    dev = mdist.init_norm_state(d, "cpu")
    for n in (5, 0, 3, 11):
        x = rng.normal(0, 2, (max(n, 1), d))[:n]
        bm = mdist.batch_moments(torch.as_tensor(x)) if n else torch.cat([torch.zeros(1), torch.zeros(d), torch.ones(d)]).double()
        b = bm.numpy()
        host = mdist.running_norm_fold(*host, b[0], b[1:1 + d], b[1 + d:])
        dev = mdist.running_norm_fold_t(*dev, bm[0], bm[1:1 + d], bm[1 + d:])
        assert float(dev[0]) == host[0]
        assert np.array_equal(dev[1].numpy(), host[1]) and np.array_equal(dev[2].numpy(), host[2])


@pytest.mark.gpu
def test_native_iteration_exchange_matches_python_path(assets):
    """msk_gpu_iteration_exchange (the C++-host form of the iteration boundary)
    equals dist.iteration_exchange bit for bit: summed stats, folded observation
    normaliser and the merged sampler; also through a 1-rank NCCL communicator."""
    import ctypes as C

    import numpy as np
    import torch

    import paper_2603_29332_b200 as pk
    import paper_2603_29332_b200.dist as pkd
    from conftest import model_paths

    mp, cp = model_paths("wb700")
    E, h = 96, 8
    envs = [pk.EnvBatch(mp, cp, E, cfg=pk.EnvConfig(episode_horizon=3, rsi=True)) for _ in range(3)]
    stats = [torch.zeros(pkd.N_STATS, dtype=torch.float64, device="cuda") for _ in envs]
    obs = [torch.empty(E, envs[0].obs_dim, device="cuda") for _ in envs]
    for g, ob in zip(envs, obs):
        g.set_eval_mode(False)
        g.reset(obs=ob)
    for it in range(2):
        for s in range(h):
            for g, st, ob in zip(envs, stats, obs):
                out = g.step(g.fill_excitations(3, it * h + s), obs=ob)
                g.rollout_stats(out["flags"], st, reward=out["reward_aux"])
                g.reset(mask=out["flags"], mask_bits=pk.FLAG_DONE)
        torch.cuda.synchronize()
        if it == 0:
            norms = [pkd.init_norm_state(envs[0].obs_dim, "cuda") for _ in envs]
            flat = [torch.cat([n[0].reshape(1), n[1], n[2]]) for n in norms[1:]]
        ref_stats, norms[0], _ = pkd.iteration_exchange(envs[0], stats[0], obs[0], norms[0], cap=h)
        s1 = envs[1].iteration_exchange(h, obs[1], stats[1], flat[0])
        comm = C.c_void_p()
        if it == 1:  # a one-rank NCCL communicator through the dlopen'ed NCCL
            class UniqueId(C.Structure):  # ncclUniqueId, passed by value
                _fields_ = [("internal", C.c_char * 128)]

            nccl = C.CDLL("libnccl.so.2")
            nccl.ncclCommInitRank.argtypes = [C.POINTER(C.c_void_p), C.c_int, UniqueId, C.c_int]
            uid = UniqueId()
            assert nccl.ncclGetUniqueId(C.byref(uid)) == 0
            assert nccl.ncclCommInitRank(C.byref(comm), 1, uid, 0) == 0
        s2 = envs[2].iteration_exchange(h, obs[2], stats[2], flat[1], nccl_comm=comm.value)
        torch.cuda.synchronize()
        for so in (s1, s2):
            assert torch.equal(so.cpu(), ref_stats.cpu())
        ref_flat = torch.cat([norms[0][0].reshape(1), norms[0][1], norms[0][2]]).cpu()
        for f in flat:
            assert torch.equal(f.cpu(), ref_flat), it
        e0 = envs[0].get_sampler().cpu()
        for g in envs[1:]:
            assert torch.equal(g.get_sampler().cpu(), e0)
        for st in stats:
            st.zero_()
        if comm.value:
            nccl.ncclCommDestroy.argtypes = [C.c_void_p]
            assert nccl.ncclCommDestroy(comm) == 0
    for g in envs:
        g.close()
