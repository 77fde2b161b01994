"""Training-loop caller: nn.Linear + ChainLoss + autograd
on the GPU, the reference demo's experiment (demo.py:81-158, SPEC.md:545 bar:
loss falls, frame accuracy >= 0.9)."""

import numpy as np
import pytest

from paper_2005_09824_b200 import train


def test_toy_graphs_are_stochastic_and_accept_their_alignments():
    rng = np.random.default_rng(1)
    corpus = train.synthesize_corpus(rng, 5, 12)
    den = train.bigram_denominator(corpus, 5)
    out = np.bincount(den.forward_from, weights=den.forward_probs, minlength=den.num_states)
    np.testing.assert_allclose((out + den.final_probs)[1:], 1.0, rtol=1e-12)
    for phones in corpus[:4]:
        tgt = train.expand_alignment(phones, 6, rng)
        num = train.numerator_graph(phones, 5)
        # the numerator accepts the alignment's length; every target pdf is on a numerator arc
        assert set(tgt.tolist()) <= set(num.forward_pdf.tolist())
        assert len(tgt) >= len(phones)


@pytest.mark.gpu
def test_train_loss_decreases_and_accuracy(cuda):
    res = train.train(num_phones=6, num_utterances=40, epochs=150, seed=0)
    assert res.losses[-1] < res.losses[0]
    assert all(np.isfinite(res.losses))
    assert res.accuracy >= 0.9, res.accuracy
    again = train.train(num_phones=6, num_utterances=40, epochs=3, seed=0)
    assert again.losses == res.losses[:3]  # deterministic kernels, fixed seed
