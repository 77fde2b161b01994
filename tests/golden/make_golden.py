"""Generate golden vectors by running the REFERENCE implementation.

Imports chainloss 0.1.0 from /root/reference/pkg/src (read-only mount, only
present in the build container) and records inputs + outputs of its public
hot-path API into tests/golden/*.npz.  The committed fixtures are what pin
the CPU oracle (oracle/) and, through it, the CUDA path; this script is
never run on the GPU box.

    PYTHONPYCACHEPREFIX=/tmp/pyc NUMBA_CACHE_DIR=/tmp/numba \
        python tests/golden/make_golden.py
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = os.environ.get("CHAINLOSS_REF_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF_SRC)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import chainloss as C  # noqa: E402
from chainloss.oracle import random_loss_instance  # noqa: E402

from paper_2005_09824_b200 import synth  # noqa: E402  (input recipe only)


def graph_fields(prefix, g):
    arcs = np.stack([g.forward_from.astype(np.float64), g.forward_to.astype(np.float64),
                     g.forward_pdf.astype(np.float64), g.forward_probs], axis=1) \
        if g.num_transitions else np.zeros((0, 4))
    bw = np.stack([g.backward_from.astype(np.float64), g.backward_to.astype(np.float64),
                   g.backward_pdf.astype(np.float64), g.backward_probs], axis=1) \
        if g.num_transitions else np.zeros((0, 4))
    # Both layouts are stored: the in-layout arc order fixes the reference's
    # summation order, which cannot be recovered from one sorted layout.
    return {f"{prefix}_arcs": arcs, f"{prefix}_bw_arcs": bw,
            f"{prefix}_meta": np.array([g.num_states, g.num_pdfs, g.initial_state], np.int64),
            f"{prefix}_finals": np.asarray(g.final_probs, np.float64)}


def record(name, batch, nums, den, leak, trellis=True):
    opts = C.FBOptions(leak_coefficient=leak)
    out = {"values": batch.values, "lengths": batch.lengths,
           "valid_batch_sizes": batch.valid_batch_sizes, "order_map": batch.order_map,
           "leak": np.float64(leak), "num_graphs": np.int64(nums.batch_size)}
    for k in range(nums.batch_size):
        out.update(graph_fields(f"num{k}", nums.graph(k)))
    out.update(graph_fields("den", den.graph(0)))
    for side, g in (("num", nums), ("den", den)):
        fb = C.forward_backward(batch, g, opts, keep_trellis=trellis)
        out[f"{side}_log_probs"] = fb.log_probs
        out[f"{side}_posteriors"] = fb.posteriors
        out[f"{side}_scale_logs"] = fb.scale_logs
        out[f"{side}_failure_frames"] = fb.failure_frames
        if trellis:
            out[f"{side}_alpha"] = fb.alpha
            out[f"{side}_beta"] = fb.beta
    try:
        res = C.chain_loss(batch, nums, den, opts)
        out.update(objective=np.float64(res.objective), loss=np.float64(res.loss), grad=res.grad,
                   per_utt=np.array(res.per_utt, np.float64), num_failed=np.int64(res.num_failed),
                   all_failed=np.int64(0))
    except RuntimeError:
        out.update(all_failed=np.int64(1))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)


def main():
    # 1. known answers (tests/test_forward_backward.py:25-29, test_loss.py:52-70)
    self_loop = C.ChainGraph([(0, 0, 0, 1.0)], 1, 1, 0, [1.0])
    two_state = C.ChainGraph([(0, 1, 0, 0.4), (0, 0, 1, 0.6), (1, 1, 0, 1.0)], 2, 2, 0, [0.0, 1.0])
    b = C.make_batch([np.zeros((2, 2))])
    record("ka_two_state", b, C.ChainGraphBatch.broadcast(two_state, 1),
           C.ChainGraphBatch.broadcast(two_state, 1), 0.0)
    b = C.make_batch([np.full((3, 1), math.log(0.5)), np.zeros((2, 1))])
    record("ka_self_loop", b, C.ChainGraphBatch.broadcast(self_loop, 2),
           C.ChainGraphBatch.broadcast(self_loop, 2), 0.0)
    num = C.ChainGraph([(0, 1, 0, 1.0), (1, 2, 1, 1.0)], 3, 2, 0, [0, 0, 1.0])
    den = C.ChainGraph([(0, 0, 0, 0.5), (0, 0, 1, 0.5)], 1, 2, 0, [1.0])
    record("ka_forced_path", C.make_batch([np.zeros((2, 2))]), C.ChainGraphBatch.from_graphs([num]),
           C.ChainGraphBatch.broadcast(den, 1), 0.0)
    chain3 = C.ChainGraph([(0, 1, 0, 1.0), (1, 2, 0, 1.0), (2, 2, 0, 0.5)], 3, 1, 0, [0, 0, 0.5])
    b = C.make_batch([np.zeros((4, 1)), np.zeros((1, 1))])
    record("ka_failure", b, C.ChainGraphBatch.broadcast(chain3, 2),
           C.ChainGraphBatch.broadcast(self_loop, 2), 0.0)
    # 2. random instances from the reference's own generator (oracle.py:195-226)
    rng = np.random.default_rng(20261017)
    leaks = [0.0, 1e-5, 1e-2]
    for k in range(24):
        batch, nums, den = random_loss_instance(rng)
        record(f"rand{k:02d}", batch, nums, den, leaks[k % 3])
    # 3. the toy config of BASELINE.json (synthetic recipe, seeds 0 and 1), no trellis
    for seed in (0, 1):
        w = synth.make_workload("toy", seed)
        batch, nums, den = w.build(C)
        record(f"toy_seed{seed}", batch, nums, den, 1e-5, trellis=False)
    print("wrote", sorted(f for f in os.listdir(HERE) if f.endswith(".npz")))


if __name__ == "__main__":
    main()
