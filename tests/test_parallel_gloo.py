"""N>1 path on CPU: world_size-2 gloo process group.

Each rank takes its LPT shard of one toy/C2-shaped batch, computes the shard's
totals {sum_ok(num - den), sum_ok T_b, #failed} (with the oracle standing in
for the GPU op, which needs a B200), all-reduces them through
``parallel.reduce_totals`` and forms the loss with ``parallel.loss_from_totals``;
the result must equal the single-process loss over the whole batch.
"""

import os
import socket

import numpy as np
import pytest

import paper_2005_09824_b200 as P
from oracle import oracle as O
from paper_2005_09824_b200 import parallel, synth


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _shard_totals(w, idx):
    """Oracle totals of the sub-batch `idx` (indices into the sorted batch)."""
    batch, nums, den = w.build(P)
    order = batch.order_map
    seqs = [w.seqs[order[i]] for i in idx]
    sub = P.make_batch(seqs)
    num_g = [nums.graph(int(i)) for i in idx]
    num_g = [num_g[j] for j in sub.order_map]
    sn = P.ChainGraphBatch.from_graphs(num_g)
    sd = P.ChainGraphBatch.broadcast(den.graph(0), len(idx))
    ref = O.chain_loss(sub, sn, sd, leak=1e-5)
    ok = [k for k in range(len(idx)) if np.isfinite(ref.per_utt[k][0] - ref.per_utt[k][1])]
    frames = float(sum(int(sub.lengths[k]) for k in ok))
    return np.array([ref.objective, frames, float(ref.num_failed)])


def _worker(rank, world, port, result_path):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = synth.make_workload("toy", seed=5, batch_size=7)
        batch, _, _ = w.build(P)
        idx = parallel.shard_of(batch.lengths, rank, world)
        tot = torch.tensor(_shard_totals(w, idx), dtype=torch.float64)
        parallel.reduce_totals(tot)
        obj, loss, nf = parallel.loss_from_totals(tot.numpy(), len(batch.lengths))
        if rank == 0:
            np.save(result_path, np.array([obj, loss, nf, len(idx)], dtype=np.float64))
    finally:
        dist.destroy_process_group()


def test_lpt_shards_partition_and_balance():
    costs = np.array([300, 299, 250, 180, 150, 150, 120, 60, 50])
    for world in (1, 2, 3, 4, 8):
        shards = parallel.lpt_shards(costs, world)
        allidx = np.sort(np.concatenate(shards))
        np.testing.assert_array_equal(allidx, np.arange(len(costs)))
        loads = [costs[s].sum() for s in shards]
        # LPT bound: max load <= (4/3 - 1/(3m)) * OPT <= 4/3 * max(mean, max item)
        assert max(loads) <= 4 / 3 * max(costs.sum() / world, costs.max()) + 1e-9
    assert parallel.lpt_shards(costs, 2)[0].tolist() == parallel.shard_of(costs, 0, 2).tolist()
    with pytest.raises(ValueError):
        parallel.lpt_shards(costs, 0)


def test_loss_from_totals_semantics():
    obj, loss, nf = parallel.loss_from_totals([-10.0, 5.0, 1.0], 3)
    assert (obj, loss, nf) == (-10.0, 2.0, 1)
    assert parallel.loss_from_totals([-10.0, 5.0, 0.0], 3, normalize_by_frames=False)[1] == 10.0
    with pytest.raises(RuntimeError, match="all 2"):
        parallel.loss_from_totals([0.0, 0.0, 2.0], 2)


def test_gloo_world2_sharded_loss_equals_single_process(tmp_path):
    import torch.multiprocessing as mp

    world = 2
    out = str(tmp_path / "r0.npy")
    mp.start_processes(_worker, args=(world, _free_port(), out), nprocs=world, join=True,
                       start_method="spawn")
    obj, loss, nf, n0 = np.load(out)
    w = synth.make_workload("toy", seed=5, batch_size=7)
    batch, nums, den = w.build(P)
    ref = O.chain_loss(batch, nums, den, leak=1e-5)
    assert abs(obj - ref.objective) <= 1e-9 * max(1.0, abs(ref.objective))
    assert abs(loss - ref.loss) <= 1e-9 * max(1.0, abs(ref.loss))
    assert int(nf) == ref.num_failed
    assert 0 < n0 < 7
