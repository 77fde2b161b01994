"""GPU parity: CUDA path (through the C-ABI) vs the pinned oracle / golden vectors.

Tolerances (BASELINE.json north_star): fp32 production path — objective
within 1e-5 relative, gradient within 1e-4 absolute.  fp64 fused path —
1e-10.  f64 parity kernels (three-phase seam) — bit-exact, since they follow
the reference operation order with no FMA contraction.
"""

import math

import numpy as np
import pytest

import paper_2005_09824_b200 as P
from golden_util import load, names
from oracle import oracle as O
from paper_2005_09824_b200 import synth

pytestmark = pytest.mark.gpu

FP32_OBJ_REL = 1e-5
FP32_GRAD_ABS = 1e-4
FP64_TOL = 1e-10


def _rel(a, b):
    return abs(a - b) / max(1.0, abs(b))


# ------------------------------------------------------------ golden vectors
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("name", names())
def test_chain_loss_vs_golden(cuda, name, precision):
    batch, nums, den, leak, z = load(name)
    opts = P.FBOptions(leak_coefficient=leak)
    if int(z["all_failed"]):
        with pytest.raises(RuntimeError, match="failed"):
            P.chain_loss(batch, nums, den, opts, precision=precision)
        return
    res = P.chain_loss(batch, nums, den, opts, precision=precision)
    otol, gtol = (FP32_OBJ_REL, FP32_GRAD_ABS) if precision == "fp32" else (FP64_TOL, FP64_TOL)
    assert _rel(res.objective, float(z["objective"])) <= otol
    assert np.abs(res.grad - z["grad"]).max() <= gtol
    assert res.num_failed == int(z["num_failed"])
    pu = np.array(res.per_utt)
    np.testing.assert_array_equal(np.isnan(pu), np.isnan(z["per_utt"]))
    ok = ~np.isnan(z["per_utt"])
    assert np.all(np.abs(pu[ok] - z["per_utt"][ok]) <= otol * np.maximum(1, np.abs(z["per_utt"][ok])))
    # normalisation (loss.py:71-72)
    assert _rel(res.loss, float(z["loss"])) <= otol


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("name", names())
def test_forward_backward_vs_golden(cuda, name, precision):
    batch, nums, den, leak, z = load(name)
    opts = P.FBOptions(leak_coefficient=leak)
    tol = 1e-5 if precision == "fp32" else FP64_TOL
    for side, g in (("num", nums), ("den", den)):
        fb = P.forward_backward(batch, g, opts, precision=precision)
        np.testing.assert_array_equal(fb.failure_frames, z[f"{side}_failure_frames"])
        ref = z[f"{side}_log_probs"]
        np.testing.assert_array_equal(np.isnan(fb.log_probs), np.isnan(ref))
        ok = ~np.isnan(ref)
        assert np.all(np.abs(fb.log_probs[ok] - ref[ok]) <= tol * np.maximum(1, np.abs(ref[ok])))
        assert np.abs(fb.posteriors - z[f"{side}_posteriors"]).max() <= (
            FP32_GRAD_ABS if precision == "fp32" else FP64_TOL)
        np.testing.assert_allclose(fb.scale_logs, z[f"{side}_scale_logs"], rtol=tol, atol=tol)


@pytest.mark.parametrize("name", [n for n in names() if not n.startswith("toy")])
def test_parity_kernels_bit_exact(cuda, name):
    """lfmmi_{forward,backward,posterior}_kernel == reference numba kernels, bitwise."""
    import torch

    from paper_2005_09824_b200 import _backend

    ext = _backend.ext()
    batch, nums, den, leak, z = load(name)
    expl, _ = O.emissions(batch.values, batch.lengths)  # reference host glue (numpy)
    dev = torch.device("cuda", 0)
    for side, g in (("num", nums), ("den", den)):
        dg = P.device_graphs(g, dev)
        pi = O.leak_distribution(g)
        B, T, D = batch.values.shape
        S = g.max_states
        a = torch.zeros((B, T + 1, S), dtype=torch.float64, device=dev)
        sc = torch.ones((B, T), dtype=torch.float64, device=dev)
        fl = torch.full((B,), -1, dtype=torch.int64, device=dev)
        ex = torch.tensor(expl, device=dev)
        ln = torch.tensor(batch.lengths, dtype=torch.int32, device=dev)
        pit = torch.tensor(pi, device=dev)
        ext.forward_kernel(dg.handle, dg.row_map, ex, ln, leak, pit, 1e-300, a, sc, fl)
        np.testing.assert_array_equal(a.cpu().numpy(), z[f"{side}_alpha"])
        np.testing.assert_array_equal(fl.cpu().numpy(), z[f"{side}_failure_frames"])
        be = torch.zeros_like(a)
        ext.backward_kernel(dg.handle, dg.row_map, ex, ln, sc, leak, pit, fl, be)
        np.testing.assert_array_equal(be.cpu().numpy(), z[f"{side}_beta"])
        gm = torch.zeros((B, T, D), dtype=torch.float64, device=dev)
        ext.posterior_kernel(dg.handle, dg.row_map, ex, ln, a, be, fl, gm)
        np.testing.assert_array_equal(gm.cpu().numpy(), z[f"{side}_posteriors"])


@pytest.mark.parametrize("name", ["ka_two_state", "rand00", "rand01", "rand02"])
def test_three_phase_api(cuda, name):
    batch, nums, den, leak, z = load(name)
    opts = P.FBOptions(leak_coefficient=leak)
    fb = P.forward_backward(batch, den, opts, keep_trellis=True)
    np.testing.assert_allclose(fb.alpha, z["den_alpha"], rtol=1e-12, atol=1e-300)
    np.testing.assert_allclose(fb.beta, z["den_beta"], rtol=1e-12, atol=1e-300)
    np.testing.assert_allclose(fb.posteriors, z["den_posteriors"], atol=1e-12)
    fwd = P.forward(batch, den, opts)
    beta = P.backward(batch, den, opts, fwd)
    gamma = P.occupation_posteriors(batch, den, fwd, beta)
    np.testing.assert_array_equal(gamma, fb.posteriors)


# ------------------------------------------------- BASELINE configs vs oracle
def _kernel_env(kernel, lib_options):
    """Kernel selection shared by the parity tests: denominator "tile" (one CTA
    per utterance), "split1"/"split2" (2-CTA split, 1 or 2 clusters), "tile1x"
    (tile kernel with one posterior slot buffer), "numtile" (numerators through
    the generic tile kernel instead of the linear-chain kernel), "smallnum" /
    "smallden" (the small-graph threshold moved either way), "g2" / "g4s" (tile
    packs with 2 / 4 lanes per state on the tile / split kernels), "ssplit" /
    "ssplit0" (L2-resident graphs on the stream split kernel, with / without
    the TMA slot ring), "tilep" (the den tile kernel as 2 persistent CTAs, several
    utterances each)."""
    if kernel == "tile":  # one CTA per utterance (no forward/backward split)
        lib_options(split=0)
    if kernel in ("split1", "split2"):  # 2-CTA split, several utterances per cluster
        lib_options(split=1)
        lib_options(split_clusters=kernel[-1])
    if kernel == "tile1x":
        lib_options(split=0, tile_xdb=0)
    if kernel == "numtile":
        lib_options(linear=0)
    if kernel == "noring":  # stream kernel reading slot rows straight from L2 (no TMA ring)
        lib_options(stream_ring=0, stream_mode="1024x1")
    if kernel == "smallnum":  # every graph <= 512 states (the hmm den too) numerator-sized
        lib_options(small_arcs=1 << 30, small_indeg=1 << 30)
    if kernel == "smallden":  # every graph on the den kernels (numerators too)
        lib_options(small_arcs=0, linear=0)
    if kernel == "g2":  # tile packs with two lanes per state (pack time), tile kernel
        lib_options(tile_g=2, split=0)
    if kernel == "g4s":  # four lanes per state, split kernel
        lib_options(tile_g=4, split=1)
    if kernel == "tilep":  # den tile kernel as 2 persistent CTAs over the in-kernel LPT
        lib_options(split=0, tile_persist=2)
    if kernel == "ssplit":  # L2-resident graphs: forward | backward stream split with its TMA ring
        lib_options(stream_mode="split", ssplit_ring=1)
    if kernel == "ssplit0":  # ... slot rows straight from L2 (the default)
        lib_options(stream_mode="split")


@pytest.mark.parametrize("kernel", ["auto", "tile", "split2", "tile1x", "numtile", "noring",
                                    "group", "smallnum", "smallden", "g2", "g4s", "ssplit",
                                    "ssplit0", "tilep"])
@pytest.mark.parametrize("config,batch_size", [("toy", None), ("wsj_mono", None), ("hmm", 24),
                                               ("wsj_biphone", 4), ("wsj_biphone", 100),
                                               ("sweep", 6)])
def test_configs_vs_oracle(cuda, config, batch_size, kernel, lib_options):
    _kernel_env(kernel, lib_options)
    if kernel == "group":  # force the generic group kernel for the denominator
        lib_options(tile=0)
        lib_options(stream=0)
    w = synth.make_workload(config, seed=3, batch_size=batch_size)
    batch, nums, den = w.build(P)
    res = P.chain_loss(batch, nums, den)
    ref = O.chain_loss(batch, nums, den, leak=1e-5)
    assert _rel(res.objective, ref.objective) <= FP32_OBJ_REL
    assert np.abs(res.grad - ref.grad).max() <= FP32_GRAD_ABS
    assert res.num_failed == ref.num_failed == 0


@pytest.mark.parametrize("kernel", ["ssplit", "stream", "stream1", "stream512", "group"])
def test_large_graph_l2_path_vs_oracle(cuda, kernel, lib_options):
    """Config 4 (20k states / 200k arcs / 2000 pdfs): the arc packs do not fit in
    shared memory.  "ssplit": the default forward | backward stream split;
    "stream": coalesced 32-state tiles streamed from L2 by one 2-CTA cluster per
    utterance (fb_stream_kernel<1024,2>); "group": the generic CSR kernel with
    alpha read back from the HBM trellis."""
    if kernel == "group":
        lib_options(stream=0)
    if kernel == "stream":
        lib_options(stream_mode="1024x2")
    if kernel == "ssplit":  # forward | backward split (fb_streamsplit_kernel)
        lib_options(stream_mode="split")
    if kernel == "stream1":  # one CTA per utterance instead of a 2-CTA cluster
        lib_options(stream_mode="1024x1")
    if kernel == "stream512":  # 2-CTA clusters of 512 threads (two per SM when they fit)
        lib_options(stream_mode="512x2")
    w = synth.make_workload("large", seed=3, batch_size=2)
    batch, nums, den = w.build(P)
    res = P.chain_loss(batch, nums, den)
    ref = O.chain_loss(batch, nums, den, leak=1e-5)
    assert _rel(res.objective, ref.objective) <= FP32_OBJ_REL
    assert np.abs(res.grad - ref.grad).max() <= FP32_GRAD_ABS
    assert res.num_failed == ref.num_failed == 0
    fb = P.forward_backward(batch, den)
    rf = O.forward_backward(batch, den, leak=1e-5)
    np.testing.assert_allclose(fb.log_probs, rf.log_probs, rtol=1e-6)
    assert np.abs(fb.posteriors - rf.posteriors).max() <= FP32_GRAD_ABS
    # deterministic: fixed-point posterior bins make the sums order-independent
    again = P.chain_loss(batch, nums, den)
    assert again.objective == res.objective
    np.testing.assert_array_equal(again.grad, res.grad)


# ------------------------------------------ size-independent properties (full C2)
@pytest.fixture(scope="module")
def c2():
    w = synth.make_workload("wsj_mono", seed=0)
    return w.build(P)


def test_c2_grad_structure(cuda, c2):
    batch, nums, den = c2
    res = P.chain_loss(batch, nums, den)
    for b in range(batch.batch_size):
        n = int(batch.lengths[b])
        assert np.abs(res.grad[b, :n].sum(axis=1)).max() <= 1e-4   # rows sum to 0
        assert np.all(res.grad[b, n:] == 0.0)                        # padding is zero
    # posteriors are distributions
    fb = P.forward_backward(batch, den)
    rs = np.concatenate([fb.posteriors[b, : batch.lengths[b]].sum(axis=1)
                         for b in range(batch.batch_size)])
    assert np.abs(rs - 1.0).max() <= 1e-4


def test_c2_deterministic_and_batch_independent(cuda, c2):
    batch, nums, den = c2
    r1 = P.chain_loss(batch, nums, den)
    r2 = P.chain_loss(batch, nums, den)
    assert r1.objective == r2.objective and np.array_equal(r1.grad, r2.grad)
    for b in (0, 77, batch.batch_size - 1):
        n = int(batch.lengths[b])
        solo = P.make_batch([batch.values[b, :n]])
        rs = P.chain_loss(solo, P.ChainGraphBatch.from_graphs([nums.graph(b)]),
                          P.ChainGraphBatch.broadcast(den.graph(0), 1))
        assert rs.per_utt[0] == r1.per_utt[b]
        assert np.array_equal(rs.grad[0], r1.grad[b, :n])


def test_c2_nan_poisoned_padding(cuda, c2):
    batch, nums, den = c2
    clean = P.chain_loss(batch, nums, den)
    v = batch.values.copy()
    for b in range(batch.batch_size):
        v[b, int(batch.lengths[b]):] = np.nan
    dirty = P.chain_loss(P.LogLikBatch(v, batch.lengths, batch.valid_batch_sizes,
                                       batch.order_map), nums, den)
    assert clean.objective == dirty.objective
    assert np.array_equal(clean.grad, dirty.grad)


def test_c2_shift_equivariance(cuda, c2):
    batch, nums, den = c2
    base = P.forward_backward(batch, den)
    v = batch.values.copy()
    v[:, 10, :] += 0.75
    shifted = P.forward_backward(P.LogLikBatch(v, batch.lengths, batch.valid_batch_sizes,
                                               batch.order_map), den)
    np.testing.assert_allclose(shifted.log_probs, base.log_probs + 0.75, rtol=1e-6)
    assert np.abs(shifted.posteriors[:, 10] - base.posteriors[:, 10]).max() <= 1e-5


# ------------------------------------------------------------- edge cases
def test_failure_semantics(cuda):
    batch, nums, den, leak, z = load("ka_failure")
    res = P.chain_loss(batch, nums, den, P.FBOptions(leak_coefficient=0.0))
    assert res.num_failed == 1
    assert np.all(res.grad[1] == 0.0)
    num_lp, den_lp = res.per_utt[1]
    assert math.isnan(num_lp) and not math.isnan(den_lp)


@pytest.mark.parametrize("late", [False, True])
@pytest.mark.parametrize("config,batch_size,kernel", [
    ("wsj_mono", 4, "auto"), ("wsj_mono", 4, "tile"), ("wsj_mono", 4, "split1"),
    ("wsj_mono", 4, "tile1x"), ("wsj_mono", 4, "numtile"),
    ("wsj_biphone", 3, "auto"), ("large", 2, "auto"), ("large", 2, "stream1")])
def test_nan_frame_fails_one_utterance_every_path(cuda, config, batch_size, kernel, late,
                                                  lib_options):
    """A NaN log-likelihood makes that utterance's column totals NaN -> it fails
    at that frame in both graphs (_kernels.py:114-118); the others are untouched
    and chain_loss excludes it (loss.py:61-69).  Covers the early-exit paths of
    the XDB tile kernel, the linear and tile numerator kernels and the 1- and
    2-CTA stream kernel."""
    _kernel_env(kernel, lib_options)
    if kernel == "stream1":
        lib_options(stream_mode="1024x1")
    w = synth.make_workload(config, seed=9, batch_size=batch_size)
    batch, nums, den = w.build(P)  # make_batch rejects non-finite input: poison afterwards
    bad = 1
    values = np.array(batch.values)
    # early frame, or one after the split kernel's midpoint (forward CTA already
    # writing posteriors, backward CTA past the barrier)
    values[bad, int(batch.lengths[bad]) - 3 if late else 5, 3] = np.nan
    batch = P.LogLikBatch(values=values, lengths=batch.lengths,
                          valid_batch_sizes=batch.valid_batch_sizes, order_map=batch.order_map)
    res = P.chain_loss(batch, nums, den)
    ref = O.chain_loss(batch, nums, den, leak=1e-5)
    assert res.num_failed == ref.num_failed == 1
    assert np.all(res.grad[bad] == 0.0)
    n, d = res.per_utt[bad]
    assert math.isnan(n) and math.isnan(d)
    assert _rel(res.objective, ref.objective) <= FP32_OBJ_REL
    assert np.abs(res.grad - ref.grad).max() <= FP32_GRAD_ABS


@pytest.mark.parametrize("mode", ["split", "splitring", "1024x1", "1024x2"])
def test_stream_kernel_short_utterances(cuda, mode, lib_options):
    """1-, 2- and 3-frame utterances through the L2-streamed kernel (biphone-sized
    denominator): prologue / epilogue edges of the register row pipeline."""
    if mode == "splitring":
        lib_options(stream_mode="split", ssplit_ring=1)
    else:
        lib_options(stream_mode=mode)
    w = synth.make_workload("wsj_biphone", seed=10, batch_size=4)
    rng = np.random.default_rng(0)
    seqs = [rng.normal(0, 2, (t, w.D)).astype(np.float32).astype(np.float64) for t in (1, 2, 3, 7)]
    batch = P.make_batch(seqs)
    den = P.ChainGraphBatch.broadcast(w.den_graph(P), 4)
    fb = P.forward_backward(batch, den)
    rf = O.forward_backward(batch, den, leak=1e-5)
    np.testing.assert_allclose(fb.log_probs, rf.log_probs, rtol=1e-6, atol=1e-6)
    assert np.abs(fb.posteriors - rf.posteriors).max() <= FP32_GRAD_ABS


@pytest.mark.parametrize("kernel", ["tile", "split1", "split2"])
def test_split_kernel_short_and_odd_utterances(cuda, kernel, lib_options):
    """1, 2, 3, 4, 7 and 300-frame utterances through the denominator tile kernels:
    midpoint h = T/2 at 0 (no backward posterior frames), odd T, and several
    utterances per cluster (split1: all in one cluster, pack bound once)."""
    _kernel_env(kernel, lib_options)
    w = synth.make_workload("wsj_mono", seed=10, batch_size=6)
    rng = np.random.default_rng(0)
    seqs = [rng.normal(0, 2, (t, w.D)).astype(np.float32).astype(np.float64)
            for t in (1, 2, 3, 4, 7, 300)]
    batch = P.make_batch(seqs)
    den = P.ChainGraphBatch.broadcast(w.den_graph(P), 6)
    fb = P.forward_backward(batch, den)
    rf = O.forward_backward(batch, den, leak=1e-5)
    np.testing.assert_allclose(fb.log_probs, rf.log_probs, rtol=1e-6, atol=1e-6)
    assert np.abs(fb.posteriors - rf.posteriors).max() <= FP32_GRAD_ABS


@pytest.mark.parametrize("kernel", ["tile", "split2"])
def test_split_kernel_bitwise_batch_independent(cuda, kernel, lib_options):
    """An utterance's result does not depend on its batch-mates or on which
    cluster / position in a cluster's list it lands (fixed reduction orders)."""
    _kernel_env(kernel, lib_options)
    w = synth.make_workload("wsj_mono", seed=11, batch_size=8)
    batch, nums, den = w.build(P)
    full = P.forward_backward(batch, den)
    sub = P.make_batch([batch.values[b, :batch.lengths[b]] for b in (2, 5)])
    part = P.forward_backward(sub, P.ChainGraphBatch.broadcast(den.graph(0), 2))
    for i, b in enumerate((2, 5)):
        assert full.log_probs[b] == part.log_probs[i]
        np.testing.assert_array_equal(full.posteriors[b, :batch.lengths[b]],
                                      part.posteriors[i, :batch.lengths[b]])


def test_custom_leak_distribution(cuda):
    w = synth.make_workload("toy", seed=5)
    batch, nums, den = w.build(P)
    rng = np.random.default_rng(1)
    pi = rng.random(den.max_states)
    pi /= pi.sum()
    res = P.chain_loss(batch, P.ChainGraphBatch.from_graphs([den.graph(0)] * batch.batch_size),
                       den, P.FBOptions(leak_coefficient=1e-2, leak_distribution=pi),
                       precision="fp64")
    assert abs(res.objective) <= 1e-9 and np.abs(res.grad).max() <= 1e-9
    fb = P.forward_backward(batch, den, P.FBOptions(leak_coefficient=1e-2, leak_distribution=pi),
                            precision="fp64")
    ref = O.forward_backward(batch, den, leak=1e-2, leak_dist=pi)
    np.testing.assert_allclose(fb.log_probs, ref.log_probs, rtol=1e-10)
    np.testing.assert_allclose(fb.posteriors, ref.posteriors, atol=1e-10)


def test_single_frame_and_ragged(cuda):
    rng = np.random.default_rng(3)
    loop = P.ChainGraph([(0, 0, 0, 0.5), (0, 0, 1, 0.5)], 1, 2, 0, [1.0])
    seqs = [rng.normal(size=(t, 2)) for t in (1, 7, 1, 3)]
    batch = P.make_batch(seqs)
    nums = P.ChainGraphBatch.from_graphs([loop] * 4)
    den = P.ChainGraphBatch.broadcast(loop, 4)
    res = P.chain_loss(batch, nums, den, precision="fp64")
    ref = O.chain_loss(batch, nums, den)
    assert abs(res.objective - ref.objective) <= 1e-12
    np.testing.assert_allclose(res.grad, ref.grad, atol=1e-12)


def test_chain_function_autograd(cuda):
    import torch

    w = synth.make_workload("toy", seed=2)
    batch, nums, den = w.build(P)
    ref = O.chain_loss(batch, nums, den, leak=1e-5)
    x = torch.tensor(batch.values, dtype=torch.float32, device="cuda", requires_grad=True)
    loss = P.ChainFunction.apply(x, torch.tensor(batch.lengths), nums, den)
    (2.0 * loss).backward()
    frames = int(batch.lengths.sum())
    assert _rel(float(loss), ref.loss) <= 1e-5
    assert np.abs(x.grad.double().cpu().numpy() + 2.0 * ref.grad / frames).max() <= 1e-5
    mod = P.ChainLoss(den.graph(0))
    l2 = mod(x, torch.tensor(batch.lengths), nums)
    assert float(l2) == float(loss)


def test_pdf_mismatch_raises(cuda):
    loop = P.ChainGraph([(0, 0, 0, 1.0)], 1, 1, 0, [1.0])
    batch = P.make_batch([np.zeros((2, 2))])
    with pytest.raises(ValueError, match="pdf dimension"):
        P.chain_loss(batch, P.ChainGraphBatch.broadcast(loop, 1), P.ChainGraphBatch.broadcast(loop, 1))


@pytest.mark.parametrize("num_group", ["32", "64", "128"])
def test_numerator_group_sizes(cuda, num_group, lib_options):
    """Numerator pass with 1, 2 or 4 warps per utterance (B < 2 x SMs default: 4)."""
    lib_options(linear=0, num_group=num_group)
    w = synth.make_workload("wsj_mono", seed=4, batch_size=6)
    batch, nums, den = w.build(P)
    res = P.chain_loss(batch, nums, den)
    ref = O.chain_loss(batch, nums, den, leak=1e-5)
    assert _rel(res.objective, ref.objective) <= FP32_OBJ_REL
    assert np.abs(res.grad - ref.grad).max() <= FP32_GRAD_ABS


@pytest.mark.parametrize("kernel", ["auto", "tile", "split2", "numtile", "stream"])
@pytest.mark.parametrize("config,batch_size", [("wsj_mono", 7), ("sweep", 5),
                                               ("wsj_biphone", 3), ("large", 2)])
def test_packed_ragged_batch_any_order(cuda, config, batch_size, kernel, lib_options):
    """Device-side batching: (sum T, D) ragged input in caller (unsorted) order,
    no padding; grad comes back in the same ragged layout."""
    import torch

    _kernel_env(kernel, lib_options)
    if kernel == "stream" and config not in ("wsj_biphone", "large"):
        pytest.skip("stream kernel is for graphs beyond shared memory")
    w = synth.make_workload(config, seed=6, batch_size=batch_size)
    batch, nums, den = w.build(P)
    ref = O.chain_loss(batch, nums, den, leak=1e-5)
    order = np.random.default_rng(0).permutation(batch.batch_size)  # arbitrary caller order
    seqs = [batch.values[b, :batch.lengths[b]] for b in order]
    dev = torch.device("cuda", 0)
    x = torch.tensor(np.concatenate(seqs), dtype=torch.float32, device=dev)
    lens = torch.tensor([len(q) for q in seqs], dtype=torch.int32, device=dev)
    num_list = [nums.graph(int(b)) for b in order]
    g, nl, dl, nf, df, tot = P.chain_loss_packed(x, lens, num_list, den.graph(0))
    tot = tot.cpu().numpy()
    assert _rel(float(tot[0]), ref.objective) <= FP32_OBJ_REL
    assert int(round(tot[1])) == int(batch.lengths.sum()) and int(round(tot[2])) == 0
    g = g.double().cpu().numpy()
    offs = np.concatenate([[0], np.cumsum([len(q) for q in seqs])])
    for k, b in enumerate(order):
        assert np.abs(g[offs[k]:offs[k + 1]] - ref.grad[b, :batch.lengths[b]]).max() <= FP32_GRAD_ABS
    nl = nl.cpu().numpy()
    for k, b in enumerate(order):
        assert _rel(nl[k], ref.per_utt[b][0]) <= 1e-5


@pytest.mark.parametrize("kernel", ["auto", "tile", "split1"])
def test_zero_length_item_fails_alone(cuda, kernel, lib_options):
    """The device APIs take lengths as a device tensor and do not read them back:
    a zero-length utterance is reported failed (NaN log-prob, failure frame 0)
    without touching memory, and the rest of the batch is unaffected."""
    import torch

    _kernel_env(kernel, lib_options)
    w = synth.make_workload("wsj_mono", seed=12, batch_size=4)
    batch, nums, den = w.build(P)
    ref = O.chain_loss(batch, nums, den, leak=1e-5)
    seqs = [batch.values[b, :batch.lengths[b]] for b in range(4)]
    dev = torch.device("cuda", 0)
    x = torch.tensor(np.concatenate(seqs), dtype=torch.float32, device=dev)
    lens = torch.tensor([len(seqs[0]), 0, *[len(q) for q in seqs[1:]]], dtype=torch.int32,
                        device=dev)
    num_list = [nums.graph(0), nums.graph(0), nums.graph(1), nums.graph(2), nums.graph(3)]
    g, nl, dl, nf, df, tot = P.chain_loss_packed(x, lens, num_list, den.graph(0))
    tot = tot.cpu().numpy()
    assert int(round(tot[2])) == 1 and int(round(tot[1])) == int(batch.lengths.sum())
    assert _rel(float(tot[0]), ref.objective) <= FP32_OBJ_REL
    assert math.isnan(float(dl[1].cpu())) and int(df[1].cpu()) == 0
    g = g.double().cpu().numpy()
    offs = np.concatenate([[0], np.cumsum([len(q) for q in seqs])])
    for b in range(4):
        assert np.abs(g[offs[b]:offs[b + 1]] - ref.grad[b, :batch.lengths[b]]).max() <= FP32_GRAD_ABS


def test_chain_function_packed_input(cuda):
    import torch

    w = synth.make_workload("wsj_mono", seed=8, batch_size=4)
    batch, nums, den = w.build(P)
    ref = O.chain_loss(batch, nums, den, leak=1e-5)
    x = torch.tensor(np.concatenate([batch.values[b, :batch.lengths[b]] for b in range(4)]),
                     dtype=torch.float32, device="cuda", requires_grad=True)
    lens = torch.tensor(batch.lengths, dtype=torch.int32)
    loss = P.ChainFunction.apply(x, lens, nums, den)
    loss.backward()
    assert _rel(float(loss.detach()), ref.loss) <= 1e-5
    frames = int(batch.lengths.sum())
    g = x.grad.double().cpu().numpy()
    exp = np.concatenate([-ref.grad[b, :batch.lengths[b]] / frames for b in range(4)])
    assert np.abs(g - exp).max() <= FP32_GRAD_ABS


def test_concurrent_streams_do_not_share_scratch(cuda):
    """Two batches on two CUDA streams at once: per-stream workspaces and
    per-thread auxiliary streams keep them independent."""
    import torch

    outs = []
    ws = [synth.make_workload("wsj_mono", seed=s, batch_size=6) for s in (11, 12)]
    built = [w.build(P) for w in ws]
    refs = [O.chain_loss(*b, leak=1e-5) for b in built]
    streams = [torch.cuda.Stream() for _ in built]
    tensors = [(torch.tensor(b[0].values, dtype=torch.float32, device="cuda"),
                torch.tensor(b[0].lengths, dtype=torch.int32, device="cuda")) for b in built]
    torch.cuda.synchronize()
    for (x, l), b, st in zip(tensors, built, streams):
        with torch.cuda.stream(st):
            outs.append(P.chain_loss_device(x, l, b[1], b[2]))
    torch.cuda.synchronize()
    for o, ref in zip(outs, refs):
        assert _rel(float(o[5][0].item()), ref.objective) <= FP32_OBJ_REL
        assert np.abs(o[0].double().cpu().numpy() - ref.grad).max() <= FP32_GRAD_ABS


def test_chain_loss_exact_workspace_concurrent_repeat(cuda):
    """Regression: numerator and denominator passes run concurrently and share one
    exactly-sized workspace; repeated calls must not overlap their regions."""
    import torch

    from paper_2005_09824_b200 import _backend

    ext = _backend.ext()
    w = synth.make_workload("wsj_mono", seed=3, batch_size=8)
    batch, nums, den = w.build(P)
    ref = O.chain_loss(batch, nums, den, leak=1e-5)
    dev = torch.device("cuda", 0)
    values = torch.tensor(batch.values, dtype=torch.float32, device=dev)
    lengths = torch.tensor(batch.lengths, dtype=torch.int32, device=dev)
    ng, dg = P.device_graphs(nums, dev), P.device_graphs(den, dev)
    B, T, D = values.shape
    tf = int(batch.lengths.sum())
    ws = torch.empty(ext.chain_loss_workspace_size(ng.handle, dg.handle, B, T, D, tf, 0),
                     dtype=torch.uint8, device=dev)
    for _ in range(3):
        grad = torch.empty_like(values)
        f64, i32 = dict(dtype=torch.float64, device=dev), dict(dtype=torch.int32, device=dev)
        nl, dl, tot = torch.empty(B, **f64), torch.empty(B, **f64), torch.empty(3, **f64)
        nf, df = torch.empty(B, **i32), torch.empty(B, **i32)
        ext.chain_loss(ng.handle, ng.row_map, dg.handle, dg.row_map, values, lengths, 1e-5,
                       1e-300, None, None, tf, ws, grad, nl, dl, nf, df, tot)
        assert np.abs(grad.double().cpu().numpy() - ref.grad).max() <= FP32_GRAD_ABS
    with pytest.raises(ValueError, match="workspace"):
        ext.chain_loss(ng.handle, ng.row_map, dg.handle, dg.row_map, values, lengths, 1e-5,
                       1e-300, None, None, tf, ws[:-1024], grad, nl, dl, nf, df, tot)


def test_chain_loss_module_ragged_steps(cuda):
    """ChainLoss over several training steps with ragged (sum T, D) input and
    a plain list of numerator graphs: batch size from input_lengths (not sum T),
    one resident denominator pack, bounded caches, loss/grad vs the oracle."""
    import torch

    from paper_2005_09824_b200 import graph as G

    w = synth.make_workload("wsj_mono", seed=41, batch_size=24)
    batch, nums, den = w.build(P)
    mod = P.ChainLoss(den.graph(0))
    packs_before = len(G._GRAPH_PACKS)
    for step, idx in enumerate([range(0, 8), range(8, 16), range(16, 24), range(4, 12)]):
        idx = list(idx)
        seqs = [batch.values[b, :batch.lengths[b]] for b in idx]
        x = torch.tensor(np.concatenate(seqs), dtype=torch.float32, device="cuda",
                         requires_grad=True)
        lens = torch.tensor([len(q) for q in seqs], dtype=torch.int32)
        loss = mod(x, lens, [nums.graph(b) for b in idx])
        loss.backward()
        sub = P.make_batch(seqs)
        sn = [nums.graph(idx[j]) for j in sub.order_map]
        ref = O.chain_loss(sub, P.ChainGraphBatch.from_graphs(sn),
                           P.ChainGraphBatch.broadcast(den.graph(0), len(idx)), leak=1e-5)
        assert _rel(float(loss.detach()), ref.loss) <= FP32_OBJ_REL, step
        g = x.grad.double().cpu().numpy()
        frames = int(sub.lengths.sum())
        offs = np.concatenate([[0], np.cumsum([len(q) for q in seqs])])
        for k, j in enumerate(sub.order_map):  # sorted item k is idx[j]
            exp = -ref.grad[k, :sub.lengths[k]] / frames
            assert np.abs(g[offs[j]:offs[j + 1]] - exp).max() <= FP32_GRAD_ABS, step
    assert len(mod._den_cache) == 1  # one batch size (8) -> one broadcast batch
    assert len(G._GRAPH_PACKS) - packs_before <= 1  # one resident den pack


def test_chain_function_all_failed_gives_zero_grad(cuda):
    """Every utterance failing (NaN input) gives loss 0 and a zero gradient,
    never NaN into the model (ADVICE: 0 * inf); chain_loss raises as the
    reference does (loss.py:63-64)."""
    import torch

    w = synth.make_workload("wsj_mono", seed=42, batch_size=3)
    batch, nums, den = w.build(P)
    x = torch.full((batch.batch_size, batch.max_length, w.D), float("nan"), device="cuda",
                   requires_grad=True)
    lens = torch.tensor(batch.lengths, dtype=torch.int32)
    loss = P.ChainFunction.apply(x, lens, nums, den)
    loss.backward()
    assert float(loss.detach()) == 0.0
    assert torch.all(x.grad == 0)
    values = np.full(batch.values.shape, np.nan)
    bad = P.LogLikBatch(values=values, lengths=batch.lengths,
                        valid_batch_sizes=batch.valid_batch_sizes, order_map=batch.order_map)
    with pytest.raises(RuntimeError, match="failed"):
        P.chain_loss(bad, nums, den)


def test_bad_lengths_fail_items_instead_of_faulting(cuda):
    """A length beyond T_max (e.g. pre-subsampling lengths) marks that item failed
    on the device instead of writing out of bounds; a wrong-sized lengths or
    numerator list raises before launch."""
    import torch

    w = synth.make_workload("wsj_mono", seed=43, batch_size=4)
    batch, nums, den = w.build(P)
    x = torch.tensor(batch.values, dtype=torch.float32, device="cuda")
    lens = torch.tensor(batch.lengths, dtype=torch.int32, device="cuda")
    lens[1] = batch.max_length + 100
    g, nl, dl, nf, df, tot = P.chain_loss_device(x, lens, nums, den)
    torch.cuda.synchronize()
    assert int(df[1]) >= 0 and int(round(float(tot[2]))) == 1
    assert torch.all(g[1] == 0)
    with pytest.raises((ValueError, RuntimeError)):
        P.chain_loss_device(x, lens[:3], nums, den)
    with pytest.raises(ValueError, match="batch has"):
        P.chain_loss_device(x[:3], lens[:3], nums, den)
