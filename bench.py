#!/usr/bin/env python3
"""Throughput benchmark: whole-body env-steps/s on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1]): the whole-body planar model
``wb700_fixed`` (80 links, 700 Hill muscles, pinned pelvis, no contacts),
4096 envs per GPU, Philox random excitations, eval mode, horizon 1000 on the
synthetic ``dance`` clip.  One "step" = one control step (10 x 2 ms
substeps) of every env, i.e. E env-steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

N > 1 runs under torchrun: every rank steps its own contiguous shard of
envs (independent units, no data-path collective -> scaling "weak");
timing is the max over ranks of the device time.

JSON line fields beyond the base contract:
  value       device-resident throughput (inputs generated on device)
  e2e         same metric through the C-ABI host-buffer call
              (msk_gpu_step_host: H2D actions, step, D2H obs/Δ/reward/flags)
  roofline    step kernel: algorithmic HBM bytes/launch ÷ its event time,
              vs MEASURED_PEAKS.json hbm_gbs; "fp32" adds the binding FP32
              roofline (algorithmic flops vs the measured FFMA peak)
  cpu_baseline the reference's own CPU path (oracle/_ref, compiled from
              /root/reference sources) on the box's host cores, bounded sample
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DEFAULT_MODEL = "wb700_fixed"

# BASELINE.json configs -> workloads.  c2 is the headline (default); the others
# are the rollout-shaped configurations (§8(d) C3-C5), measured on request.
CONFIGS = {
    "c2": dict(model="wb700_fixed", envs=4096, eval=True, rsi=False, horizon=1000, reward_mode=0, disc=None,
               exchange=0, desc="wb700_fixed: 80 links, 700 muscles, no contacts, eval mode, random excitations"),
    "c3": dict(model="wb700_fixed", envs=8192, eval=True, rsi=False, horizon=1000, reward_mode=0, disc=None,
               exchange=8, desc="wb700_fixed, 8192 envs/GPU (65536 on 8 GPUs), rollout-stats allgather + "
                            "ordered sampler/obs-norm merge every 8 control steps"),
    "c4": dict(model="wb700", envs=16384, eval=False, rsi=True, horizon=250, reward_mode=2, disc=(256, 7),
               exchange=8, desc="wb700 (floating root, 10 contact spheres), dance clip, training mode (RSI, "
                            "adaptive sampler, 0.5 m termination, auto-reset), fused tracking reward "
                            "-log(1-D(delta)) (D: Mlp W=256 seed 7 on tcgen05) + ImitationPower 0.05, "
                            "allgather every 8 steps"),
    "c2g": dict(model="wb700_general", envs=4096, eval=True, rsi=False, horizon=1000, reward_mode=0, disc=None,
                exchange=0, desc="c2 with the generic-segment whole-body variant wb700_general: 46% of the 700 "
                             "muscles span non-adjacent links (generic world-frame muscle path)"),
    "c5": dict(model="wb700_slow", envs=8192, eval=False, rsi=True, horizon=250, reward_mode=2, disc=None,
               exchange=8, desc="stress: wb700 with contacts, tau_act=0.05 / tau_deact=0.20 for all muscles, "
                            "training mode with mid-batch resets, allgather every 8 steps"),
}
CLIPS = {"wb700_fixed": "wb700_fixed_dance", "wb700": "wb700_dance", "arm2_m6": "arm2_m6_sine",
         "walker5_m16": "walker5_m16_sine", "wb700_slow": "wb700_dance", "wb700_general": "wb700_fixed_dance"}


def ensure_assets():
    d = os.path.join(ROOT, "assets", "generated")
    need = ["wb700_fixed.json", "wb700_fixed_dance.csv", "wb700.json", "wb700_dance.csv", "arm2_m6.json",
            "wb700_general.json", "wb700_slow.json"]
    if not all(os.path.exists(os.path.join(d, n)) for n in need):
        from tools.gen_assets import generate
        generate(d)
    return d


def model_files(name):
    d = ensure_assets()
    return os.path.join(d, name + ".json"), os.path.join(d, CLIPS[name] + ".csv")


# ----------------------------------------------------------------------------
# algorithmic cost model
# ----------------------------------------------------------------------------
def cost_model(model_json):
    """Algorithmic HBM bytes and FLOPs per env-step, from the model file."""
    with open(model_json) as f:
        js = json.load(f)
    floating = js["root"] == "floating"
    joints = js.get("joints", [])
    mus = js.get("muscles", [])
    vias = [vp for m in mus for vp in m["via_points"]]
    starts = [0]
    for m in mus:
        starts.append(starts[-1] + len(m["via_points"]))
    spheres = js.get("contacts", {}).get("spheres", [])
    d = {"floating": floating, "joint_parent": [int(j["parent"]) for j in joints], "via_link": [int(v[0]) for v in vias],
         "m_via_start": starts, "n_spheres": len(spheres), "sphere_link": [int(s["link"]) for s in spheres]}
    nj, nl, nm, nk = len(joints), len(js["links"]), len(mus), len(js.get("key_bodies", []))
    nq = (3 if floating else 0) + nj
    obs_dim = 3 * nq + 6 * nk + 4 * nm
    ddim = 3 + nj + 2 * nk
    bytes_per = 4 * (nm + 2 * (2 * nq + 2 * nm) + obs_dim + ddim + 3)
    # tree depths
    fc = 1 if d["floating"] else 0
    parent = [-1] * nl
    for j in range(nj):
        parent[fc + j] = int(d["joint_parent"][j])
    depth = [0] * nl
    for l in range(nl):
        depth[l] = depth[parent[l]] + 1 if parent[l] >= 0 else (0 if d["floating"] and l == 0 else 1)
    V = len(d["via_link"])
    S = V - nm
    # segment/joint pairs of J_m^T F (joints strictly between a segment's links)
    def path(l):
        out = set()
        while l >= fc:
            out.add(l - fc)
            l = parent[l]
        return out
    P = 0
    for m in range(nm):
        a, b = d["m_via_start"][m], d["m_via_start"][m + 1]
        for v in range(a + 1, b):
            la, lb = int(d["via_link"][v - 1]), int(d["via_link"][v])
            if la != lb:
                P += len(path(la) ^ path(lb))
    ns = d["n_spheres"]
    f_sub = (12 * nl + 8 * V + 7 * S + 41 * nm + 2 * S + 6 * P + 8 * nl + sum(21 + 12 * dl for dl in depth)
             + 4 * nj + sum(35 + 5 * depth[int(s)] for s in d["sphere_link"])
             + sum(2 * dl + 2.5 * dl * dl for dl in depth) + sum(dl * dl + 4 * dl for dl in depth) + 4 * nq)
    f_ctrl = 12 * nl + 30 * nk + nj
    flops_per = 10 * f_sub + f_ctrl
    return dict(bytes_per_env_step=int(bytes_per), flops_per_env_step=float(flops_per), n_pairs=P, n_via=V,
                obs_dim=obs_dim, delta_dim=ddim, nq=nq, nm=nm, ns=ns)


# ----------------------------------------------------------------------------
def clocks_sampler(stop, out, gpu_index):
    q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    try:
        p = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "20",
                              "-i", str(gpu_index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
    except FileNotFoundError:
        return
    while not stop.is_set():
        line = p.stdout.readline()
        if not line:
            break
        out.append((time.monotonic(), line.strip()))
    p.terminate()


def summarize_clocks(lines, t0=None, t1=None):
    """Median SM clock and throttle reasons over the samples taken in [t0, t1]."""
    lines = [ln for t, ln in lines if (t0 is None or t >= t0) and (t1 is None or t <= t1)]
    sm, mx, reasons = [], 0.0, set()
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    for ln in lines:
        f = [x.strip() for x in ln.split(",")]
        if len(f) < 9:
            continue
        try:
            sm.append(float(f[1]))
            mx = max(mx, float(f[2]))
        except ValueError:
            continue
        for n, v in zip(names, f[5:9]):
            if v.lower().startswith("active"):
                reasons.add(n)
    sm.sort()
    return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx or None, "reasons": sorted(reasons),
            "samples": len(sm)}


# ----------------------------------------------------------------------------
def host_link_bound(dev, h2d_bytes, d2h_bytes, envs, step_ms, e2e_value):
    """The e2e loop's host-link ceiling: one step's pinned H2D and D2H copies
    timed alone (CUDA events, best of 6, the two directions concurrent on two
    streams as in the pipelined loop); `frac` = e2e / that bound."""
    import torch

    hi = torch.empty(h2d_bytes, dtype=torch.uint8, pin_memory=True)
    hd = torch.empty(h2d_bytes, dtype=torch.uint8, device=dev)
    ho = torch.empty(d2h_bytes, dtype=torch.uint8, pin_memory=True)
    do = torch.empty(d2h_bytes, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def timed(s, dst, src):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            dst.copy_(src, non_blocking=True)
            e1.record(s)
        return e0, e1

    best = [1e30, 1e30, 1e30]
    for _ in range(6):
        torch.cuda.synchronize(dev)
        a = timed(s1, hd, hi)
        torch.cuda.synchronize(dev)
        b = timed(s2, ho, do)
        torch.cuda.synchronize(dev)
        c = timed(s1, hd, hi), timed(s2, ho, do)  # both directions at once
        torch.cuda.synchronize(dev)
        best[0] = min(best[0], a[0].elapsed_time(a[1]))
        best[1] = min(best[1], b[0].elapsed_time(b[1]))
        best[2] = min(best[2], max(c[0][0].elapsed_time(c[0][1]), c[1][0].elapsed_time(c[1][1])))
    h2d_ms, d2h_ms, both_ms = best
    bound = envs / (both_ms * 1e-3)
    return {"h2d_gbs": h2d_bytes / (h2d_ms * 1e6), "d2h_gbs": d2h_bytes / (d2h_ms * 1e6),
            "duplex_ms": both_ms, "device_step_ms": step_ms,
            "bound": bound, "frac": e2e_value / bound,
            "note": "link ceiling = envs / one step's H2D + D2H copies run concurrently (pinned, CUDA events); "
                    "the e2e loop overlaps env groups' copies with other groups' steps, so the device step "
                    "is hidden while it is shorter than the copies"}


def cpu_model():
    """Host CPU model name and logical core count (for the CPU-arm lines)."""
    name = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    name = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"model": name, "logical_cpus": os.cpu_count()}


def ref_build(fast):
    return ("reference sources (oracle/_ref) g++ -O3 -march=x86-64-v3 -ffp-contract=fast, eager Eigen shim"
            if fast else "reference sources (oracle/_ref) g++ -O2 -march=x86-64-v3 -ffp-contract=off, eager Eigen shim")


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU path (oracle/_ref) on the host cores."""
    if rank != 0:
        return
    from oracle.ref import REF_FAST_SO, RefBatch, env_config

    mp, cp = model_files(args.model)
    C = args.C
    threads = args.cpu_threads or os.cpu_count() or 1
    n_envs = args.ref_envs or 8 * threads  # E_cpu = 8 x cores
    cfg = env_config(episode_horizon=C["horizon"], rsi=C["rsi"])
    fast = os.path.exists(REF_FAST_SO)  # the -O3 / FMA build of the same reference sources
    b = RefBatch(mp, cp, n_envs, cfg=cfg, threads=threads, reward_mode=C["reward_mode"], fast=fast)
    b.set_eval_mode(C["eval"])
    if C["disc"]:  # Env::step(action, fn) with the reference's own Mlp as fn (same θ as the GPU arm)
        import paper_2603_29332_b200 as pk

        b.set_discriminator(pk.mlp_init(b.delta_dim, C["disc"][0], C["disc"][1]), C["disc"][0])
    b.reset()
    for _ in range(args.warmup):
        b.bench(1)
    secs, steps = b.bench(args.steps)
    v = steps / secs
    line = {"metric": "env-steps/sec (700-muscle whole-body)", "value": v, "unit": "env-steps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (Philox excitations, generated dance clip)", "impl": "reference",
            "config": {"workload": f"{args.config}: {C['desc']} (CPU sample"
                                   + ("; D(Δ) reward by the reference's own Mlp::forward_one)" if C["disc"] else ")"),
                       "config": args.config, "envs": n_envs,
                       "parallelism": f"{threads} host threads (ThreadPool::parallel_chunks)"},
            "cpu_baseline": {"value": v, "unit": "env-steps/s", "cores": threads, "kind": "reference",
                             "sample": f"{n_envs} envs x {args.steps} control steps ({secs:.1f} s)",
                             "cpu": cpu_model(), "build": ref_build(fast)},
            "e2e": {"value": v, "unit": "env-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline_sample(args):
    """Bounded sample (~10-20 s) of the reference CPU path for the cpu_baseline key."""
    from oracle.ref import REF_FAST_SO, RefBatch, env_config

    mp, cp = model_files(args.model)
    C = args.C
    threads = args.cpu_threads or os.cpu_count() or 1
    n_envs = 8 * threads  # E_cpu = 8 x cores
    fast = os.path.exists(REF_FAST_SO)
    b = RefBatch(mp, cp, n_envs, cfg=env_config(episode_horizon=C["horizon"], rsi=C["rsi"]), threads=threads,
                 reward_mode=C["reward_mode"], fast=fast)
    b.set_eval_mode(C["eval"])
    if C["disc"]:
        import paper_2603_29332_b200 as pk

        b.set_discriminator(pk.mlp_init(b.delta_dim, C["disc"][0], C["disc"][1]), C["disc"][0])
    b.reset()
    b.bench(1)
    secs, steps = b.bench(1)
    per_step = secs
    k = max(1, min(5000, int(args.cpu_seconds / max(per_step, 1e-3))))
    secs, steps = b.bench(k)
    return {"value": steps / secs, "unit": "env-steps/s", "cores": threads, "kind": "reference",
            "sample": f"{n_envs} envs x {k} control steps of {args.model} ({secs:.1f} s)", "cpu": cpu_model(),
            "build": ref_build(fast)}


def self_launch(n):
    """Re-runs this command under torch.distributed.run with n ranks on this node
    (127.0.0.1 rendezvous); returns its exit code (rank 0 prints the JSON line)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    print(f"[bench] launching {n} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.run(cmd).returncode


def run_dry(args, rank, world):
    """--dry-run: the multi-rank plumbing on CPU (gloo), no GPU: every rank builds a
    synthetic iteration block (outcomes of its env shard, stats, observation
    moments), all-gathers it and applies the rank-ordered merge (dist.py, the
    same code the GPU ranks run); rank 0 prints one JSON line with what it saw."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2603_29332_b200.dist as pkd

    if world > 1:
        dist.init_process_group("gloo")
    E, cap, D = 64, 8, 12
    g = np.random.default_rng(100 + rank)
    bins = torch.tensor(g.integers(0, 10, (E, cap)), dtype=torch.int16)
    failed = torch.tensor(g.integers(0, 2, (E, cap)), dtype=torch.uint8)
    counts = torch.tensor(g.integers(0, cap + 1, E), dtype=torch.int32)
    stats = torch.tensor([float(E), 1.0 * rank, 0.0, 0.0, 0.0, 0.0, 0.0], dtype=torch.float64)
    obs = torch.tensor(g.normal(rank, 1.0, (E, D)))
    norm = pkd.batch_moments(obs)
    blocks = pkd.exchange(pkd.pack_block(bins, failed, counts, stats, norm, D))
    st, (cnt, mean, var), ema = pkd.merged_iteration(blocks, E, cap, D, (0.0, np.zeros(D), np.ones(D)),
                                                      np.zeros(10), 0.99)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "ranks_in_exchange": len(blocks),
                          "env_steps_merged": float(st[0]), "rank_sum": float(st[1]), "norm_count": float(cnt),
                          "sampler_ema": [float(x) for x in ema]}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS), help="BASELINE.json workload")
    ap.add_argument("--envs", type=int, default=0, help="envs per GPU (default: the config's)")
    ap.add_argument("--model", default="", help="override the config's model")
    ap.add_argument("--cpu-threads", type=int, default=0)
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--ref-envs", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-groups", type=int, default=4, help="env groups (contexts) in the e2e host-buffer loop")
    ap.add_argument("--rollout", action="store_true", help="record every step into the on-device rollout buffer "
                    "and run GAE at each iteration boundary")
    ap.add_argument("--policy-width", type=int, default=0,
                    help="actions from the on-device flow policy of this hidden width (0: Philox excitations)")
    ap.add_argument("--disc-train", default="", choices=["", "fp32", "bf16"],
                    help="train the reward discriminator on the device once per rollout iteration (needs --rollout "
                         "and a config with D): one Adam step on the iteration's h*E Delta rows, then publish")
    ap.add_argument("--dry-run", action="store_true", help="CPU-only check of the multi-rank exchange plumbing "
                    "(gloo; no GPU): self-launch, all_gather and the rank-ordered merge")
    ap.add_argument("--e2e-steps", type=int, default=0, help="timed end-to-end iterations (default max(100, steps))")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    C = dict(CONFIGS[args.config])
    args.model = args.model or C["model"]
    args.envs = args.envs or C["envs"]
    args.C = C
    if C["exchange"]:  # the first iteration boundary (allocations) falls inside the warm-up
        args.warmup = max(args.warmup, C["exchange"] + 1)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `bench.py --gpus N` launches its own N ranks (one process per GPU) when no
        # launcher did: the same torchrun command line the driver uses
        raise SystemExit(self_launch(args.gpus))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")

    if args.dry_run:
        run_dry(args, rank, world)
        return
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    import paper_2603_29332_b200 as pk
    import paper_2603_29332_b200.dist as pkd

    if local >= torch.cuda.device_count():
        raise SystemExit(f"bench.py: rank {rank} needs cuda:{local} but this node has {torch.cuda.device_count()} GPUs")
    torch.cuda.set_device(local)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        t = torch.ones(1, device="cuda")
        dist.all_reduce(t)  # communicator up: every rank contributes
        comm = {"backend": "nccl", "nranks": dist.get_world_size(), "all_reduce_check": float(t.item())}
        if rank == 0:
            print(f"[bench] NCCL communicator nranks={comm['nranks']} (all_reduce of ones = {t.item():.0f})",
                  file=sys.stderr, flush=True)
    mp, cp = model_files(args.model)
    E = args.envs
    cfg = pk.EnvConfig(episode_horizon=C["horizon"], rsi=C["rsi"])
    rcfg = pk.RewardConfig(mode=C["reward_mode"])
    env = pk.EnvBatch(mp, cp, E, cfg=cfg, reward=rcfg, global_env_offset=rank * E)
    env.set_eval_mode(C["eval"])
    dev = env.device
    stream = torch.cuda.current_stream(dev)
    actions = torch.empty(E, env.nm, device=dev)
    obs = torch.empty(E, env.obs_dim, device=dev)
    delta = torch.empty(E, env.delta_dim, device=dev)
    raux = torch.empty(E, device=dev)
    reward = torch.zeros(E, device=dev) if C["disc"] else None
    flags = torch.zeros(E, dtype=torch.uint8, device=dev)
    if C["disc"]:  # frozen D = Mlp(delta_dim, W, 1, Sigmoid) initialised as Mlp(shape, seed) (nn.cpp:16-38)
        width, dseed = C["disc"]
        env.set_discriminator(pk.mlp_init(env.delta_dim, width, dseed), width)
    env.reset(obs=obs)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)  # 256 MB > 126 MB L2
    seed = 0x5EED
    norm_state = pkd.init_norm_state(env.obs_dim, dev)
    # rollout stats (dist.py N_STATS): steps, sum r, sum r^2, sum episode length, episodes, failures, divergences
    stats = torch.zeros(pkd.N_STATS, dtype=torch.float64, device=dev)

    policy = None
    if args.policy_width:  # on-device policy: Gaussian π0 + 20-step flow ODE (frozen random-init Mlps)
        W = args.policy_width
        policy = pk.Policy(env.obs_dim, env.nm, W, pk.mlp_init(env.obs_dim, W, 1, n_out=env.nm, final_init_scale=0.01),
                           [-1.0] * env.nm, pk.mlp_init(5 + env.obs_dim + env.nm, W, 2, n_out=env.nm,
                                                        final_init_scale=0.01),
                           n_ode=20, dt_ode=0.05, max_envs=E, head_offset=0.5)

    rollout = None
    if args.rollout:  # on-device rollout buffer of h = 8 steps + GAE at each iteration boundary
        h_ro = C["exchange"] or 8
        rollout = pk.Rollout(E, h_ro, env.obs_dim, env.nm, env.delta_dim)
        ro_a0 = torch.empty(E, env.nm, device=dev)
        ro_lp = torch.zeros(E, device=dev)
        ro_v = torch.zeros(E, device=dev)  # no critic on this path: V = 0
    trainer = None
    if args.disc_train:  # SPEC.md:412-421 on the rollout's Δ, lr 3e-5, λ = 10
        if not (rollout is not None and C["disc"]):
            raise SystemExit("--disc-train needs --rollout and a config with a discriminator (c4)")
        width, dseed = C["disc"]
        trainer = pk.DiscTrainer(env.delta_dim, width, pk.mlp_init(env.delta_dim, width, dseed), lr=3e-5,
                                 grad_penalty=10.0, max_rows=rollout.h * E, math=1 if args.disc_train == "bf16" else 0)
        ro_delta = rollout.field(7, env.delta_dim)

    mom_acc = None  # observation moments of the current iteration (h x E observations)

    def one_step(s, ev=None):
        """One control step of the workload; ev (optional) = [start, actions, step, stats,
        exchange, reset] events recorded at the phase boundaries."""
        nonlocal norm_state, mom_acc
        if rollout is not None:  # the observation the action is taken from
            rollout.record(s % rollout.h, obs=obs)
        if C["exchange"]:  # the normaliser sees every observation the policy acts on
            if mom_acc is None:  # count 0: the first fold takes the batch moments exactly
                mom_acc = torch.zeros(1 + 2 * env.obs_dim, dtype=torch.float64, device=dev)
            env.obs_moments_fold(obs, mom_acc)
        if policy is not None:
            policy.sample(obs, explore=True, seed=seed, step=s, global_env_offset=rank * E, actions=actions,
                          a0=ro_a0 if rollout is not None else None, logprob=ro_lp if rollout is not None else None,
                          graph=True)
        else:
            env.fill_excitations(seed, s, actions)
        if ev:
            ev[1].record(stream)
        env.step(actions, obs=obs, delta=delta, reward_aux=raux, flags=flags, reward=reward)
        if ev:
            ev[2].record(stream)
        if rollout is not None:
            rollout.record(s % rollout.h, a0=ro_a0 if policy is not None else None, actions=actions,
                           logprob=ro_lp, reward=reward if reward is not None else raux, flags=flags, value=ro_v,
                           delta=delta)
            if (s + 1) % rollout.h == 0:
                rollout.gae(ro_v, gamma=0.99, lam=0.95, normalize=True)
        if C["exchange"]:
            env.rollout_stats(flags, stats, reward=reward if reward is not None else raux)
        if ev:
            ev[3].record(stream)
        if C["exchange"] and (s + 1) % C["exchange"] == 0:  # iteration boundary (h control steps)
            _, norm_state, _ = pkd.iteration_exchange(env, stats, obs, norm_state, cap=C["exchange"], moments=mom_acc)
            stats.zero_()
            mom_acc = None
        if trainer is not None and (s + 1) % rollout.h == 0:  # D update on the iteration's Δ, then publish
            trainer.step(ro_delta)
            trainer.publish(env)
        if ev:
            ev[4].record(stream)
        env.reset(mask=flags, mask_bits=pk.FLAG_DONE, obs=obs if (policy is not None or C["exchange"]) else None)
        if ev:
            ev[5].record(stream)

    for s in range(args.warmup):
        one_step(s)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk_lines, stop = [], threading.Event()
    th = threading.Thread(target=clocks_sampler, args=(stop, clk_lines, local), daemon=True)
    th.start()
    time.sleep(0.3)
    # timed region: per-step CUDA events (L2 flushed between steps, outside the events)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(args.steps)]
    n0 = env.launch_count
    torch.cuda.synchronize()
    t_loop0 = time.monotonic()
    for s in range(args.steps):
        flush.zero_()
        evs[s][0].record(stream)
        one_step(args.warmup + s, evs[s])
    torch.cuda.synchronize()
    t_loop1 = time.monotonic()
    launches = env.launch_count - n0
    stop.set()
    ms = sum(e[0].elapsed_time(e[5]) for e in evs)
    kms = sum(e[1].elapsed_time(e[2]) for e in evs) / args.steps
    phases = {name: sum(e[i].elapsed_time(e[i + 1]) for e in evs) / args.steps
              for i, name in enumerate(["actions", "step", "rollout_stats", "iteration_exchange", "reset"])}
    t = torch.tensor([ms, kms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, kms = float(t[0]), float(t[1])
    value = E * world * args.steps / (ms * 1e-3)

    # e2e through the C-ABI host-buffer call (pinned host in/out)
    e2e = None
    if not args.no_e2e:
        # End to end through the host-buffer C ABI, as an RL harness drives it:
        # the envs of this GPU split into `groups` contexts (env groups), each
        # stepped with msk_gpu_step_host_async + msk_gpu_host_wait, so one
        # group's PCIe transfers overlap the other group's step.  Every step
        # copies that step's actions in (pinned) and its obs/Δ/reward/flags out.
        groups = max(1, args.e2e_groups)
        eg = E // groups
        envs_e = [pk.EnvBatch(mp, cp, eg, cfg=cfg, reward=rcfg, global_env_offset=rank * E + g * eg)
                  for g in range(groups)]
        bufs = []
        for ge in envs_e:
            ge.set_eval_mode(C["eval"])
            ge.set_host_pipeline(1, 1)  # one chunk per group: the groups themselves pipeline
            if C["disc"]:
                ge.set_discriminator(pk.mlp_init(ge.delta_dim, C["disc"][0], C["disc"][1]), C["disc"][0])
            ge.reset()
            a_dev = ge.fill_excitations(seed, 12345)
            bufs.append(dict(
                a=a_dev.cpu().pin_memory(), o=torch.empty(eg, ge.obs_dim, pin_memory=True),
                d=torch.empty(eg, ge.delta_dim, pin_memory=True), r=torch.empty(eg, pin_memory=True),
                f=torch.zeros(eg, dtype=torch.uint8, pin_memory=True),
                w=torch.empty(eg, pin_memory=True) if C["disc"] else None))

        def issue(g):
            b = bufs[g]
            envs_e[g].step_host_async(b["a"], b["o"], b["d"], b["r"], b["f"], reward_host=b["w"])

        def collect(g):  # wait for the group's results (now in host memory), auto-reset done envs
            envs_e[g].host_wait()
            f = bufs[g]["f"]
            if f.any():  # the reset runs on torch's stream: wait for it alone (not for the other groups)
                envs_e[g].reset(mask=f.to(dev, non_blocking=True), mask_bits=pk.FLAG_DONE)
                torch.cuda.current_stream(dev).synchronize()

        for _ in range(2):
            for g in range(groups):
                issue(g)
            for g in range(groups):
                collect(g)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        k2 = args.e2e_steps or max(100, args.steps)
        t0 = time.perf_counter()
        for g in range(groups):
            issue(g)
        for it in range(k2):
            for g in range(groups):
                collect(g)
                if it + 1 < k2:
                    issue(g)
        tt = time.perf_counter() - t0
        tv = torch.tensor([tt], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tv, op=dist.ReduceOp.MAX)
        e2e = {"value": eg * groups * world * k2 / float(tv[0]), "unit": "env-steps/s",
               "h2d_bytes_per_step": E * env.nm * 4,
               "d2h_bytes_per_step": E * (env.obs_dim + env.delta_dim + 1 + (1 if C["disc"] else 0)) * 4 + E,
               "api": f"msk_gpu_step_host_async/host_wait, {groups} env groups of {eg}"}
        for ge in envs_e:
            ge.close()
        e2e["link"] = host_link_bound(dev, e2e["h2d_bytes_per_step"], e2e["d2h_bytes_per_step"], E * world, ms / args.steps, e2e["value"])

    disc = None
    if C["disc"]:  # the tensor-core kernel alone on this step's Δ (for its own roofline)
        width = C["disc"][0]
        rr = torch.empty(E, device=dev)
        for _ in range(3):
            env.discriminator_reward(delta, reward=rr)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 50
        e0.record(stream)
        for _ in range(reps):
            env.discriminator_reward(delta, reward=rr)
        e1.record(stream)
        torch.cuda.synchronize()
        dms = e0.elapsed_time(e1) / reps
        flops = 2.0 * (env.delta_dim * width + 2 * width * width + width) * E
        disc = {"kernel": "disc_reward_precise_kernel (tcgen05 kind::f16, split-bf16 operands hi+lo, 3 MMAs per "
                          "product, fp32 TMEM accumulate: fp32-class, the default mode)",
                "width": width, "ms": dms, "flops_per_launch": flops,
                "note": "flops counted once per product (the algorithmic count); the tensor cores execute 3x"}

    if rank == 0:
        cm = cost_model(mp)
        peaks = {}
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
                peaks = json.load(f)
        except OSError:
            pass
        hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
        achieved_gbs = cm["bytes_per_env_step"] * E / (kms * 1e-3) / 1e9
        fp32 = None
        try:
            import paper_2603_29332_b200.diag as diag
            pk_tf = diag.fp32_peak_tflops()
            ach_tf = cm["flops_per_env_step"] * E / (kms * 1e-3) / 1e12
            fp32 = {"achieved": ach_tf, "peak": pk_tf, "unit": "TFLOP/s", "frac": ach_tf / pk_tf,
                    "flops_per_env_step": cm["flops_per_env_step"], "peak_source": "measured FFMA probe"}
        except Exception as ex:  # pragma: no cover
            fp32 = {"error": str(ex)}
        traffic, issue = None, None
        tp = os.path.join(ROOT, "profiles", "step_kernel_traffic.json")
        if os.path.exists(tp) and args.config == "c2" and args.model == C["model"] and E == C["envs"]:
            with open(tp) as f:  # the committed ncu --set full capture of this kernel on this workload
                prof = json.load(f)
            traffic = prof.get("bytes_per_launch")
            met = prof.get("metrics", {})
            try:  # the binding resource: instruction issue slots (SURVEY §8(d) "FP32-issue bound")
                inst = float(met["smsp__inst_executed.sum"][0])
                issue = {"issue_slot_frac": float(met["smsp__issue_active.avg.pct_of_peak_sustained_active"][0]) / 100,
                         "warp_inst_per_env_substep": inst / (E * 10),
                         "l1tex_frac": float(met["l1tex__throughput.avg.pct_of_peak_sustained_active"][0]) / 100,
                         "fma_pipe_frac": float(met["sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"][0])
                         / 100, "source": "ncu --set full, profiles/step_kernel_traffic.json"}
            except (KeyError, ValueError):
                issue = None
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            try:
                cpu = cpu_baseline_sample(args)
            except Exception as ex:
                cpu = {"error": str(ex)}
        line = {
            "metric": "env-steps/sec (700-muscle whole-body)", "value": value, "unit": "env-steps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32 (f64 q/qdot, sampler)",
            "data": "synthetic (Philox excitations, generated dance clip, random-init model)",
            "config": {"workload": C["desc"] if args.model == C["model"] else f"{args.config} with model {args.model}",
                       "config": args.config, "envs_per_gpu": E, "global_envs": E * world,
                       "clip": CLIPS[args.model], "parallelism": f"env shards x{world}",
                       "actions": (f"on-device policy: Gaussian pi0 + 20-step flow ODE, Mlp width {args.policy_width} "
                                   "(tcgen05 GEMMs, CUDA graph)") if args.policy_width else "Philox excitations",
                       "rollout": "on-device buffer + GAE" if args.rollout else None,
                       **({"disc_train": f"one Adam step per iteration on h*E Delta rows ({args.disc_train} tcgen05 "
                                         "GEMMs) + device publish, inside the iteration_exchange phase"}
                          if args.disc_train else {}),
                       "l2": "flushed between timed steps"},
            "roofline": {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved_gbs / hbm_peak, "traffic": traffic,
                         "bytes_per_env_step": cm["bytes_per_env_step"], "step_kernel_ms": kms,
                         "note": "path is FP32-issue bound (SURVEY §8(d)); see fp32 and issue", "fp32": fp32,
                         **({"issue": issue} if issue else {})},
            "cpu_baseline": cpu,
            "e2e": e2e,
            **({"disc_kernel": dict(disc, achieved_tflops=disc["flops_per_launch"] / (disc["ms"] * 1e-3) / 1e12,
                                    peak_tflops=float(peaks.get("bf16_tflops", 2250.0)),
                                    frac=disc["flops_per_launch"] / (disc["ms"] * 1e-3) / 1e12
                                    / float(peaks.get("bf16_tflops", 2250.0)), bound="tensor")}
               if disc else {}),
            "gpu_launches": launches,
            **({"comm": comm} if comm else {}),
            "phases_ms_per_step": phases,
            "clocks": summarize_clocks(clk_lines, t_loop0, t_loop1),
        }
        print(json.dumps(line), flush=True)
    env.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
