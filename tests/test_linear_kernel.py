"""GPU parity of the linear-chain numerator kernel (csrc/lfmmi_linear.cu).

The reference's numerators are linear chains (toy_builder.py:218-265); the
dispatcher runs them on ``fb_linear_kernel<K>`` (lane l owns states
[l K, l K + K)).  Checked against the oracle (pinned to the reference) for
every K, leak on/off/large, D a multiple of 4 or not, every posterior write
mode, failure (an utterance too short for its transcript, a NaN frame) and
the per-utterance fast path (lists of graphs -> lfmmi_graphs_create_linear).
"""

import math

import numpy as np
import pytest

import paper_2005_09824_b200 as P
from oracle import oracle as O
from paper_2005_09824_b200 import synth

pytestmark = pytest.mark.gpu

GRAD_ABS = 1e-4


def _numerators(rng, n_phones_list, D):
    graphs = []
    for n in n_phones_list:
        phones = rng.integers(0, D // 2, n).tolist()
        arcs, S, finals = synth.numerator_arcs(phones, D // 2)
        graphs.append(P.ChainGraph(arcs, S, D, 0, finals))
    return graphs


def _batch(rng, lengths, D):
    seqs = [rng.normal(0, 2, (int(t), D)).astype(np.float32).astype(np.float64) for t in lengths]
    return P.make_batch(seqs)


@pytest.mark.parametrize("leak", [0.0, 1e-5, 0.1])
@pytest.mark.parametrize("D", [10, 84, 87, 2000])
@pytest.mark.parametrize("S_max", [20, 60, 120, 250, 500])
def test_linear_forward_backward_vs_oracle(cuda, S_max, D, leak):
    if leak == 0.0 and S_max > 120:
        # Leak-free, a transcript of hundreds of phones drives the scaled beta of
        # the states the forward pass deems unlikely past fp32's range (the
        # reference runs in fp64); every fp32 path shares this limit, and the
        # leak (1e-5 by default) bounds it.  Covered up to S = 120 here.
        pytest.skip("leak-free recursion beyond fp32 range at S > 120")
    rng = np.random.default_rng(S_max * 7 + D)
    B = 5
    n_phones = [S_max - 1, max(1, S_max // 2), 1, max(1, S_max // 3), max(1, S_max - 5)]
    # T >= #phones.  Without the leak, only paths that advance on most frames
    # reach the final state when T < ~2n, and its share of the normalised column
    # (a binomial tail, ~e-60 at T = 1.4 n) is below fp32's range while fp64
    # keeps it: leak-free utterances get T in [2n, 3n] (the leak, 1e-5 by
    # default, puts lambda / S on every state each frame and removes the issue).
    if leak > 0:
        lengths = [n + int(rng.integers(0, 2 * n + 3)) for n in n_phones]
    else:
        lengths = [2 * n + int(rng.integers(0, n + 3)) for n in n_phones]
    batch = _batch(rng, lengths, D)
    graphs = _numerators(rng, n_phones, D)
    nums = P.ChainGraphBatch.from_graphs([graphs[i] for i in batch.order_map])
    opts = P.FBOptions(leak_coefficient=leak)
    fb = P.forward_backward(batch, nums, opts)
    kern = str(P._backend.ext().last_kernel())
    assert kern.startswith("fb_linear_kernel"), kern
    rf = O.forward_backward(batch, nums, leak=leak)
    np.testing.assert_array_equal(fb.failure_frames, rf.failure_frames)
    _close(fb.log_probs, rf.log_probs)
    np.testing.assert_allclose(fb.scale_logs, rf.scale_logs, rtol=1e-5, atol=1e-5)
    assert np.abs(fb.posteriors - rf.posteriors).max() <= GRAD_ABS


def _close(a, b, rel=1e-5):
    """|a - b| <= rel * max(1, |b|) elementwise (the objective tolerance)."""
    a, b = np.asarray(a), np.asarray(b)
    assert np.all(np.abs(a - b) <= rel * np.maximum(1.0, np.abs(b))), (a, b)


def test_linear_failures_match_reference(cuda):
    """Leak-free, an utterance shorter than its transcript cannot reach the
    final state (column total 0 at its last frame: fail at T-1); a NaN frame
    fails its utterance at that frame (either leak).  The others are untouched."""
    rng = np.random.default_rng(3)
    D = 84
    n_phones = [40, 40, 40, 40]
    lengths = [100, 30, 100, 90]          # item 1: 30 frames < 40 phones
    batch = _batch(rng, lengths, D)
    values = np.array(batch.values)
    k = int(np.flatnonzero(batch.order_map == 3)[0])
    values[k, 17, 5] = np.nan             # item 3: NaN in frame 17
    batch = P.LogLikBatch(values=values, lengths=batch.lengths,
                          valid_batch_sizes=batch.valid_batch_sizes, order_map=batch.order_map)
    graphs = _numerators(rng, n_phones, D)
    nums = P.ChainGraphBatch.from_graphs([graphs[i] for i in batch.order_map])
    fb = P.forward_backward(batch, nums, P.FBOptions(leak_coefficient=0.0))
    rf = O.forward_backward(batch, nums, leak=0.0)
    np.testing.assert_array_equal(fb.failure_frames, rf.failure_frames)
    assert (fb.failure_frames >= 0).sum() == 2
    ok = rf.failure_frames < 0
    _close(fb.log_probs[ok], rf.log_probs[ok])
    assert np.all(np.isnan(fb.log_probs[~ok]))
    assert np.all(fb.posteriors[~ok] == 0.0)
    assert np.abs(fb.posteriors - rf.posteriors).max() <= GRAD_ABS
    np.testing.assert_allclose(fb.scale_logs[ok], rf.scale_logs[ok], rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("mode", [0, 1, 2, 3])  # WRITE, SUBTRACT, ADD, NEGATE
def test_linear_posterior_write_modes(cuda, mode):
    import torch

    rng = np.random.default_rng(5)
    D = 84
    batch = _batch(rng, [120, 80, 150], D)
    graphs = _numerators(rng, [30, 20, 45], D)
    nums = P.ChainGraphBatch.from_graphs([graphs[i] for i in batch.order_map])
    rf = O.forward_backward(batch, nums, leak=1e-5)
    dev = torch.device("cuda", 0)
    x = torch.tensor(batch.values, dtype=torch.float32, device=dev)
    lens = torch.tensor(batch.lengths, dtype=torch.int32, device=dev)
    base = torch.tensor(rng.normal(size=batch.values.shape), dtype=torch.float32, device=dev)
    post, lp, fail, _ = P.forward_backward_device(x, lens, nums, posteriors=base.clone(), mode=mode)
    g = rf.posteriors
    b0 = base.double().cpu().numpy()
    want = {0: g, 1: b0 - g, 2: b0 + g, 3: -g}[mode]
    valid = np.arange(batch.max_length)[None, :] < batch.lengths[:, None]
    if mode in (0, 3):  # writing modes zero the padded rows
        want = np.where(valid[:, :, None], want, 0.0)
    assert np.abs(post.double().cpu().numpy() - want).max() <= GRAD_ABS


def test_linear_graph_lists_fast_path(cuda):
    """chain_loss_packed with a plain list of numerator graphs assembles the
    batch from per-utterance records (no padded batch, no graph-pack build):
    same results as the padded reference path."""
    import torch

    w = synth.make_workload("wsj_mono", seed=21, batch_size=16)
    batch, nums, den = w.build(P)
    ref = O.chain_loss(batch, nums, den, leak=1e-5)
    dev = torch.device("cuda", 0)
    x = torch.tensor(np.concatenate([batch.values[b, :batch.lengths[b]] for b in range(16)]),
                     dtype=torch.float32, device=dev)
    lens = torch.tensor(batch.lengths, dtype=torch.int32, device=dev)
    graphs = [nums.graph(b) for b in range(16)]
    g, nl, dl, nf, df, tot = P.chain_loss_packed(x, lens, graphs, den.graph(0))
    assert isinstance(P.device_graphs(graphs, dev, linear_ok=True), P.graph.LinearDeviceGraphs)
    tot = tot.cpu().numpy()
    assert abs(tot[0] - ref.objective) <= 1e-5 * max(1.0, abs(ref.objective))
    g = g.double().cpu().numpy()
    offs = np.concatenate([[0], np.cumsum(batch.lengths)])
    for b in range(16):
        assert np.abs(g[offs[b]:offs[b + 1]] - ref.grad[b, :batch.lengths[b]]).max() <= GRAD_ABS
    nl = nl.cpu().numpy()
    for b in range(16):
        assert abs(nl[b] - ref.per_utt[b][0]) <= 1e-5 * max(1.0, abs(ref.per_utt[b][0]))


def test_linear_bitwise_batch_independent(cuda):
    """Fixed-point posterior bins and per-warp recursion: an utterance's result
    does not depend on its batch-mates."""
    rng = np.random.default_rng(8)
    D = 84
    lengths = [200, 150, 260, 90, 120]
    batch = _batch(rng, lengths, D)
    graphs = _numerators(rng, [60, 45, 80, 25, 35], D)
    nums = P.ChainGraphBatch.from_graphs([graphs[i] for i in batch.order_map])
    full = P.forward_backward(batch, nums)
    sub = P.make_batch([batch.values[b, :batch.lengths[b]] for b in (1, 3)])
    part = P.forward_backward(sub, P.ChainGraphBatch.from_graphs([nums.graph(1), nums.graph(3)]))
    for k, b in enumerate((1, 3)):
        T = int(batch.lengths[b])
        assert part.log_probs[k] == full.log_probs[b]
        np.testing.assert_array_equal(part.posteriors[k, :T], full.posteriors[b, :T])


def test_linear_disabled_falls_back_to_tile(cuda, lib_options):
    lib_options(linear=0)
    rng = np.random.default_rng(9)
    batch = _batch(rng, [60, 40], 84)
    graphs = _numerators(rng, [15, 10], 84)
    nums = P.ChainGraphBatch.from_graphs([graphs[i] for i in batch.order_map])
    fb = P.forward_backward(batch, nums)
    assert "tile" in str(P._backend.ext().last_kernel())
    rf = O.forward_backward(batch, nums, leak=1e-5)
    _close(fb.log_probs, rf.log_probs)
    assert not math.isnan(float(fb.log_probs[0]))


@pytest.mark.parametrize("split", [1, 0])
@pytest.mark.parametrize("config,batch_size,leak", [("toy", None, 1e-5), ("wsj_mono", 16, 1e-5),
                                                    ("wsj_mono", 9, 0.0), ("wsj_mono", 9, 0.1),
                                                    ("sweep", 6, 1e-5), ("wsj_biphone", 4, 1e-5)])
def test_linear_split_in_chain_loss_vs_oracle(cuda, lib_options, config, batch_size, leak, split):
    """The chain-loss numerator pass (emissions pre-pass): forward | backward warps
    meeting at the midpoint, posteriors pre-normalised by the kappa recursion
    (split = 1, the default), or one warp doing both (split = 0).  Sweep mixes
    K <= 8 utterances (split kernel) with K = 16 ones (single-warp launch).
    emit = 2: the pre-pass also for the biphone den (whose L2-streamed kernels do
    not consume it, so `auto` skips it there)."""
    lib_options(linear_split=split, emit=2)
    w = synth.make_workload(config, seed=31, batch_size=batch_size)
    batch, nums, den = w.build(P)
    opts = P.FBOptions(leak_coefficient=leak)
    res = P.chain_loss(batch, nums, den, opts)
    ref = O.chain_loss(batch, nums, den, leak=leak)
    assert abs(res.objective - ref.objective) <= 1e-5 * max(1.0, abs(ref.objective))
    assert np.abs(res.grad - ref.grad).max() <= GRAD_ABS
    for (a, _), (c, _) in zip(res.per_utt, ref.per_utt):
        assert abs(a - c) <= 1e-5 * max(1.0, abs(c))
    kern = str(P._backend.ext().last_kernel())
    assert ("split" in kern) == bool(split), kern


def test_linear_split_bitwise_batch_independent(cuda):
    """Per-utterance K and fixed orders: a numerator's log-probability and
    gradient rows do not depend on its batch-mates in the split kernel either."""
    import torch

    w = synth.make_workload("wsj_mono", seed=33, batch_size=10)
    batch, nums, den = w.build(P)
    dev = torch.device("cuda", 0)
    seqs = [batch.values[b, :batch.lengths[b]] for b in range(10)]

    def run(idx):
        x = torch.tensor(np.concatenate([seqs[i] for i in idx]), dtype=torch.float32, device=dev)
        ln = torch.tensor([len(seqs[i]) for i in idx], dtype=torch.int32, device=dev)
        g, nl, _, _, _, _ = P.chain_loss_packed(x, ln, [nums.graph(i) for i in idx], den.graph(0))
        return g.cpu().numpy(), nl.cpu().numpy()

    gf, nf = run(list(range(10)))
    gs, ns = run([3, 7])
    offs = np.concatenate([[0], np.cumsum([len(q) for q in seqs])])
    assert ns[0] == nf[3] and ns[1] == nf[7]
    np.testing.assert_array_equal(gs[:len(seqs[3])], gf[offs[3]:offs[4]])


@pytest.mark.parametrize("k16w", [2, 1])
@pytest.mark.parametrize("leak", [1e-5, 0.1])
def test_linear_k16_class_vs_oracle(cuda, lib_options, k16w, leak):
    """Numerators with S > 256 (the K = 16 class, sweep's long utterances): two
    warps per direction (64 lanes x 8 states, the default) or one (32 x 16),
    next to K <= 8 utterances in the same batch."""
    lib_options(linear_k16w=k16w)
    w = synth.make_workload("sweep", seed=5, batch_size=6)
    rng = np.random.default_rng(17)
    T = [1500, 1210, 800, 300, 905, 61]
    w.seqs = [rng.normal(0.0, 2.0, size=(t, w.D)).astype(np.float32).astype(np.float64) for t in T]
    w.lengths = np.asarray(T, dtype=np.int64)
    w.num_phones = [rng.integers(0, w.D // 2, max(1, t // 3)).tolist() for t in T]
    batch, nums, den = w.build(P)
    assert nums.max_states > 256
    opts = P.FBOptions(leak_coefficient=leak)
    res = P.chain_loss(batch, nums, den, opts)
    ref = O.chain_loss(batch, nums, den, leak=leak)
    assert abs(res.objective - ref.objective) <= 1e-5 * max(1.0, abs(ref.objective))
    assert np.abs(res.grad - ref.grad).max() <= GRAD_ABS
    for (a, _), (c, _) in zip(res.per_utt, ref.per_utt):
        assert abs(a - c) <= 1e-5 * max(1.0, abs(c))
