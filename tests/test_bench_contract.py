"""bench.py's driver contract on CPU: the reference arm (`--impl reference`)
prints one JSON line with the keys the driver reads, for the headline config,
and non-zero ranks under torchrun print nothing."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libmsk_ref.so")


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="reference build oracle/_ref absent")
def test_reference_arm_json_line():
    env = dict(os.environ, RANK="0", WORLD_SIZE="1")
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "3",
                          "--ref-envs", "4", "--cpu-threads", "4"], cwd=ROOT, capture_output=True, text=True,
                         timeout=600, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["config"]["config"] == "c2" and d["cpu_baseline"]["kind"] == "reference"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["unit"] == d["unit"]
    assert d["warmup"] >= 3


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="reference build oracle/_ref absent")
def test_reference_arm_nonzero_rank_is_silent():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup",
                          "3"],
                         cwd=ROOT, capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0 and not [l for l in out.stdout.splitlines() if l.startswith("{")]


def _json_line(out):
    return [json.loads(ln) for ln in out.splitlines() if ln.startswith("{")]


def test_bench_gpus_2_self_launches_two_ranks_dry_run():
    """`bench.py --gpus 2` without a launcher starts two ranks itself (torchrun,
    127.0.0.1); --dry-run runs the per-iteration exchange over gloo on CPU: both
    ranks' blocks reach rank 0 and the rank-ordered merge equals a single-process
    merge of the two blocks in rank order."""
    import numpy as np
    import torch

    import paper_2603_29332_b200.dist as pkd

    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_line(r.stdout)
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    d = lines[0]
    assert d["n_gpus"] == 2 and d["ranks_in_exchange"] == 2
    assert d["env_steps_merged"] == 128.0 and d["rank_sum"] == 1.0 and d["norm_count"] == 128.0
    # the same blocks merged in one process, rank order
    bins, failed, counts = [], [], []
    for rank in range(2):
        g = np.random.default_rng(100 + rank)
        bins.append(g.integers(0, 10, (64, 8)))
        failed.append(g.integers(0, 2, (64, 8)))
        counts.append(g.integers(0, 9, 64))
    ema = pkd.merge_outcomes_host(np.zeros(10), torch.tensor(np.concatenate(bins)), torch.tensor(np.concatenate(failed)),
                                  torch.tensor(np.concatenate(counts)), 0.99)
    assert d["sampler_ema"] == [float(x) for x in ema]


def test_bench_refuses_a_world_size_mismatch():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                       capture_output=True, text=True, timeout=120, env=env, cwd=ROOT)
    assert r.returncode != 0 and "WORLD_SIZE=1" in (r.stderr + r.stdout)
