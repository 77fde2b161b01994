"""The reference's own orchestration on the GPU kernel seam.

``paper_2005_09824_b200.kernel_seam.install(chainloss)`` rebinds
``chainloss._kernels.{forward,backward,posterior}_kernel`` (the numba seam,
/root/reference/pkg/src/chainloss/_kernels.py:54-224) to the C-ABI parity
kernels through ctypes — exactly the binding INTEGRATION.md shows.  The
unmodified reference (installed in ``baseline/_ref``, which travels to the GPU
box) then runs its ``chain_loss`` / ``forward_backward`` with our kernels and
is compared against itself on numba.  The parity kernels keep the
reference's operation order, so the results are expected bit-for-bit.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def chainloss():
    if not os.path.isdir(os.path.join(REF, "chainloss")):
        pytest.skip("reference not installed in baseline/_ref")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_lfmmi")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import chainloss as C

    return C


def test_seam_symbols_exported():
    from paper_2005_09824_b200 import kernel_seam

    for name in ("forward_kernel", "backward_kernel", "posterior_kernel", "install",
                 "uninstall"):
        assert callable(getattr(kernel_seam, name))


@pytest.mark.gpu
def test_reference_chain_loss_through_gpu_seam(cuda, chainloss):
    from paper_2005_09824_b200 import kernel_seam

    C = chainloss
    rng = np.random.default_rng(2024)
    cases = [C.oracle.random_loss_instance(rng) for _ in range(40)]
    cpu = [C.chain_loss(*c) for c in cases]
    kernel_seam.install(C)
    try:
        gpu = [C.chain_loss(*c) for c in cases]
    finally:
        kernel_seam.uninstall(C)
    for a, b in zip(cpu, gpu):
        assert a.objective == b.objective
        assert a.num_failed == b.num_failed
        np.testing.assert_array_equal(a.grad, b.grad)
        assert a.per_utt == b.per_utt


@pytest.mark.gpu
@pytest.mark.parametrize("leak", [0.0, 1e-5, 1e-2])
def test_reference_forward_backward_trellis_through_gpu_seam(cuda, chainloss, leak):
    from paper_2005_09824_b200 import kernel_seam

    C = chainloss
    rng = np.random.default_rng(7)
    batch, nums, den = C.oracle.random_loss_instance(rng, max_batch=3, max_frames=8, max_pdfs=5)
    opts = C.FBOptions(leak_coefficient=leak)
    ref = [C.forward_backward(batch, g, opts, keep_trellis=True) for g in (nums, den)]
    kernel_seam.install(C)
    try:
        got = [C.forward_backward(batch, g, opts, keep_trellis=True) for g in (nums, den)]
    finally:
        kernel_seam.uninstall(C)
    for a, b in zip(ref, got):
        np.testing.assert_array_equal(a.log_probs, b.log_probs)
        np.testing.assert_array_equal(a.alpha, b.alpha)
        np.testing.assert_array_equal(a.beta, b.beta)
        np.testing.assert_array_equal(a.posteriors, b.posteriors)
        np.testing.assert_array_equal(a.failure_frames, b.failure_frames)


@pytest.mark.gpu
def test_reference_c2_slice_through_gpu_seam(cuda, chainloss):
    """WSJ-mono-shaped denominator (S=1000, I=10000, D=84), 4 utterances."""
    from paper_2005_09824_b200 import kernel_seam, synth

    C = chainloss
    w = synth.make_workload("wsj_mono", seed=1, batch_size=4)
    batch, nums, den = w.build(C)
    ref = C.chain_loss(batch, nums, den)
    kernel_seam.install(C)
    try:
        got = C.chain_loss(batch, nums, den)
    finally:
        kernel_seam.uninstall(C)
    assert got.objective == ref.objective
    np.testing.assert_array_equal(got.grad, ref.grad)
