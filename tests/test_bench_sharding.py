"""bench.py's multi-GPU host logic on CPU: the sweep config's single global
batch is LPT-sharded so every rank derives the same disjoint cover (no input
scatter), weak-scaling configs give each rank its own seeded batch, and the
ideal-speed-up bound is SURVEY.md §8(e)'s formula."""

import argparse
import importlib.util
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _args(config, batch):
    return argparse.Namespace(config=config, batch=batch)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_sweep_shards_cover_the_global_batch(bench, world):
    args = _args("sweep", 48)
    shards = [bench.rank_workload(args, r, world) for r in range(world)]
    g, scaling, info = shards[0]
    assert scaling == "strong"
    assert info["global_B"] == 48
    seen = []
    for w, _, inf in shards:
        assert inf == info  # every rank derives the same global facts
        seen.extend(int(t) for t in w.lengths)
    total = sum(sum(int(t) for t in w.lengths) for w, _, _ in shards)
    assert total == info["global_frames"]
    assert len(seen) == 48
    assert info["shard_cost_imbalance"] < 1.25


def test_weak_configs_seed_per_rank(bench):
    a0 = bench.rank_workload(_args("toy", None), 0, 2)
    a1 = bench.rank_workload(_args("toy", None), 1, 2)
    assert a0[1] == a1[1] == "weak" and a0[2] is None
    assert not np.array_equal(a0[0].seqs[0][:2], a1[0].seqs[0][:2])


def test_ideal_bound(bench):
    T = np.full(1024, 800)
    assert bench.ideal_bound(T, 1) == 1.0
    # sum T / (G * 148) = 691 < T_max = 800 at G = 8: bound by the longest utterance
    assert bench.ideal_bound(T, 8) == pytest.approx((1024 * 800 / 148) / 800)
    assert bench.ideal_bound(T, 2) == pytest.approx(2.0)
