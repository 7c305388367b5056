"""Multi-GPU exchange of the env-stepper.

Envs are independent, so the data path has NO collective: rank r steps global
envs [r*E, (r+1)*E) (seeds base + global index, so any sharding gives
identical per-env results).  Once per rollout iteration every rank packs a
fixed-size block

    outcome bins  int16 [E, cap]   (Env::drain_episode_outcomes, env.cpp:200-204)
    outcome failed uint8 [E, cap]
    outcome counts int32 [E]

(cap = the iteration's h control steps: an env ends at most one episode per
step, so h slots hold every outcome of an iteration; 3 bytes per slot)
    rollout stats  float64 [7]     (n_steps, Σr, Σr², Σ episode length, episodes, failures, divergences)
    obs moments    float64 [1 + 2 D]  (count, mean[D], population var[D] of this rank's batch)

into one byte buffer and ``all_gather``s it (NCCL over NVLink on GPUs, gloo in
the CPU tests).  Every rank then applies the SAME rank-ordered merge:

* outcomes are recorded into ONE replicated adaptive sampler in global env
  order, then time order (``AdaptiveSampler::record``, env.cpp:34-37 — the
  "order-fixed reduction" of SPEC.md:296; on GPU: ``EnvBatch.merge_outcomes``);
* rollout stats are summed in rank order (f64);
* observation moments are folded in rank order with ``RunningNorm::update``'s
  parallel-variance formula (nn.cpp:246-270).

So all ranks end the iteration with bit-identical sampler and normaliser
state without an all-reduce.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

N_STATS = 7


def block_layout(n_envs: int, cap: int, obs_dim: int):
    """Byte offsets of the per-rank block."""
    sizes = [("bins", 2 * n_envs * cap), ("failed", n_envs * cap), ("counts", 4 * n_envs),
             ("stats", 8 * N_STATS), ("norm", 8 * (1 + 2 * obs_dim))]
    off, lay = 0, {}
    for name, nbytes in sizes:
        pad = (-off) % 8
        off += pad
        lay[name] = (off, nbytes)
        off += nbytes
    return lay, off


def pack_block(bins, failed, counts, stats, norm, obs_dim):
    """Packs one rank's iteration results into a uint8 tensor (same device as bins)."""
    n, cap = bins.shape
    lay, total = block_layout(n, cap, obs_dim)
    buf = torch.zeros(total, dtype=torch.uint8, device=bins.device)

    def put(name, t):
        o, nb = lay[name]
        buf[o:o + nb] = t.contiguous().view(torch.uint8).reshape(-1)

    put("bins", bins.to(torch.int16))
    put("failed", failed.to(torch.uint8))
    put("counts", counts.to(torch.int32))
    put("stats", stats.to(torch.float64))
    put("norm", norm.to(torch.float64))
    return buf


def unpack_block(buf, n_envs, cap, obs_dim):
    lay, _ = block_layout(n_envs, cap, obs_dim)

    def get(name, dtype, shape):
        o, nb = lay[name]
        return buf[o:o + nb].view(dtype).reshape(shape)

    return dict(bins=get("bins", torch.int16, (n_envs, cap)), failed=get("failed", torch.uint8, (n_envs, cap)),
                counts=get("counts", torch.int32, (n_envs,)), stats=get("stats", torch.float64, (N_STATS,)),
                norm=get("norm", torch.float64, (1 + 2 * obs_dim,)))


def batch_moments(obs: torch.Tensor):
    """(count, mean, population var) of an [n, D] batch, f64 (RunningNorm::update's batch terms)."""
    x = obs.to(torch.float64)
    n = x.shape[0]
    mean = x.mean(0)
    var = ((x - mean) ** 2).sum(0) / max(n, 1)
    return torch.cat([torch.tensor([float(n)], dtype=torch.float64, device=x.device), mean, var])


def running_norm_fold(count, mean, var, n, bmean, bvar):
    """RunningNorm::update (nn.cpp:246-270) given a batch's (n, mean, var); numpy f64."""
    if n == 0:
        return count, mean, var
    if count == 0.0:
        return float(n), bmean.copy(), bvar.copy()
    tot = count + n
    delta = bmean - mean
    var = (var * count + bvar * n + delta * delta * (count * n / tot)) / tot
    mean = mean + delta * (n / tot)
    return tot, mean, var


def merge_outcomes_host(ema, bins, failed, counts, decay):
    """Reference-order merge on the host (strict IEEE f64, no FMA contraction).

    Mirrors msk_gpu_merge_outcomes: env order, then time order, into one
    sampler EMA (AdaptiveSampler::record, env.cpp:34-37)."""
    ema = [float(x) for x in ema]
    bins_n = np.asarray(bins)
    fail_n = np.asarray(failed)
    cnt_n = np.asarray(counts)
    cap = bins_n.shape[1]
    for g in range(bins_n.shape[0]):
        for i in range(min(int(cnt_n[g]), cap)):
            b = int(bins_n[g, i])
            if 0 <= b < len(ema):
                ema[b] = decay * ema[b] + (1.0 - decay) * (1.0 if fail_n[g, i] else 0.0)
    return np.array(ema)


def exchange(block: torch.Tensor, group=None):
    """all_gather of the fixed-size per-rank block; returns the list in rank order."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return [block]
    out = [torch.empty_like(block) for _ in range(world)]
    dist.all_gather(out, block, group=group)
    return out


def running_norm_fold_t(count, mean, var, n, bmean, bvar):
    """running_norm_fold on device tensors (0-d count / n), no host sync; the
    count == 0 branch takes the batch moments exactly, as nn.cpp:257-262."""
    tot = count + n
    delta = bmean - mean
    var_m = (var * count + bvar * n + delta * delta * (count * n / tot)) / tot
    mean_m = mean + delta * (n / tot)
    first = count == 0.0
    keep = n == 0.0
    mean = torch.where(keep, mean, torch.where(first, bmean, mean_m))
    var = torch.where(keep, var, torch.where(first, bvar, var_m))
    return torch.where(keep, count, tot), mean, var


def init_norm_state(obs_dim, device):
    """RunningNorm(dim) on the device: count 0, mean 0, var 1 (nn.hpp:88-93)."""
    return (torch.zeros((), dtype=torch.float64, device=device), torch.zeros(obs_dim, dtype=torch.float64, device=device),
            torch.ones(obs_dim, dtype=torch.float64, device=device))


def merged_iteration(blocks, n_envs, cap, obs_dim, norm_state, ema, decay, merge_on_device=None):
    """Applies the rank-ordered merge to the gathered blocks.

    Returns (stats_sum [7], norm_state, ema or None).  When ``merge_on_device``
    (an EnvBatch) is given, the outcome merge runs on the GPU
    (msk_gpu_merge_outcomes) and ``ema`` is ignored."""
    parts = [unpack_block(b, n_envs, cap, obs_dim) for b in blocks]
    count, mean, var = norm_state
    on_device = torch.is_tensor(mean)
    stats = torch.zeros(N_STATS, dtype=torch.float64, device=mean.device if on_device else "cpu")
    for p in parts:  # rank order
        if on_device:  # fold on the device: no host round trip at the iteration boundary
            stats += p["stats"]
            nm = p["norm"]
            count, mean, var = running_norm_fold_t(count, mean, var, nm[0], nm[1:1 + obs_dim], nm[1 + obs_dim:])
        else:
            stats += p["stats"].cpu()
            nm = p["norm"].cpu().numpy()
            count, mean, var = running_norm_fold(count, mean, var, nm[0], nm[1:1 + obs_dim], nm[1 + obs_dim:])
    bins = torch.cat([p["bins"] for p in parts]).to(torch.int32)
    failed = torch.cat([p["failed"] for p in parts])
    counts = torch.cat([p["counts"] for p in parts])
    if merge_on_device is not None:
        merge_on_device.merge_outcomes(bins, failed.to(torch.uint8), counts)
        new_ema = None
    else:
        new_ema = merge_outcomes_host(ema, bins.cpu(), failed.cpu(), counts.cpu(), decay)
    return stats, (count, mean, var), new_ema


def fold_moments(acc, m, obs_dim):
    """Chan / RunningNorm::update merge (nn.cpp:246-270) of two moment vectors
    [n, mean[D], var[D]] (f64 device tensors, no host sync): the iteration's
    observation moments accumulate step by step over its h x E observations."""
    if acc is None:
        return m.clone()
    c, mean, var = running_norm_fold_t(acc[0], acc[1:1 + obs_dim], acc[1 + obs_dim:], m[0], m[1:1 + obs_dim],
                                       m[1 + obs_dim:])
    return torch.cat([c.reshape(1), mean, var])


def iteration_exchange(env, rollout_stats: torch.Tensor, obs_batch, norm_state, cap=64, group=None, moments=None):
    """One iteration boundary on a GPU rank: drain, pack, all_gather, ordered merge (device sampler).
    The observation moments are those of ``obs_batch`` [n x D] or, when given,
    ``moments`` [n, mean[D], var[D]] (e.g. folded over the iteration's h steps)."""
    bins, failed, counts = env.drain_outcomes(cap)
    norm = moments if moments is not None else env.obs_moments(obs_batch)  # native f64 column moments
    block = pack_block(bins, failed, counts, rollout_stats.to(bins.device), norm, env.obs_dim)
    blocks = exchange(block, group)
    return merged_iteration(blocks, env.n, cap, env.obs_dim, norm_state, None, env.cfg.adaptive_decay,
                            merge_on_device=env)
