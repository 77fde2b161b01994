"""Training-loop caller of the LF-MMI loss.

The reference's ``train_demo`` (/root/reference/pkg/src/chainloss/demo.py:81-158)
trains a single affine map from synthetic per-frame features to pdf scores by
full-batch gradient ascent on the sequence objective, with numpy gradients.
This module runs the same kind of experiment the way a PyTorch user would:
an ``nn.Linear`` on the GPU, the paper's :class:`~.loss.ChainLoss` module as
the criterion, ``loss.backward()`` and a torch optimizer — so the whole path
(nnet output → fused LF-MMI kernels → gradient w.r.t. the nnet output →
autograd into the weights) is exercised end to end.

Graphs follow the reference's toy conventions (toy_builder.py:41-64): phone
``q`` has an entry pdf ``2q`` and a loop pdf ``2q+1``; numerators are linear
phone chains (toy_builder.py:218-265 without LM), the denominator is a
phone-loop over an add-k smoothed bigram estimated from the training
transcripts (toy_builder.py:117-215, 268-310 restated compactly here).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from .forward_backward import FBOptions
from .graph import ChainGraph
from .synth import numerator_arcs

__all__ = ["TrainResult", "synthesize_corpus", "expand_alignment", "bigram_denominator",
           "numerator_graph", "train"]


@dataclass
class TrainResult:
    losses: list = field(default_factory=list)   # loss entering each epoch
    accuracy: float = 0.0                        # frame argmax accuracy after training
    total_frames: int = 0
    frames_per_s: float = 0.0                    # training steps (fwd + LF-MMI + bwd + update)


def synthesize_corpus(rng: np.random.Generator, num_phones: int, num_utterances: int,
                      max_words: int = 3, max_word_length: int = 4) -> list:
    """Random word-segmented phone transcripts (flattened to phone lists)."""
    corpus = []
    for _ in range(num_utterances):
        phones = []
        for _ in range(int(rng.integers(1, max_words + 1))):
            phones += [int(p) for p in rng.integers(0, num_phones, int(rng.integers(1, max_word_length + 1)))]
        corpus.append(phones)
    return corpus


def expand_alignment(phones, frames_per_phone: int, rng: np.random.Generator) -> np.ndarray:
    """Frame-level pdf targets: each phone's entry pdf once, then its loop pdf."""
    jitter = max(1, frames_per_phone // 3)
    out = []
    for p in phones:
        dur = max(1, frames_per_phone + int(rng.integers(-jitter, jitter + 1)))
        out.append(2 * p)
        out.extend([2 * p + 1] * (dur - 1))
    return np.asarray(out, dtype=np.int64)


def numerator_graph(phones, num_phones: int, self_loop: float = 0.5) -> ChainGraph:
    arcs, n, finals = numerator_arcs(phones, num_phones, self_loop)
    return ChainGraph(arcs, n, 2 * num_phones, 0, finals)


def bigram_denominator(corpus, num_phones: int, self_loop: float = 0.5,
                       smoothing: float = 0.1) -> ChainGraph:
    """Phone-loop denominator over an add-k bigram of the transcripts.

    State 0 starts; state q+1 is phone q's loop state (self-loop ``rho`` on the
    loop pdf, exit mass ``1-rho`` split by P(q'|q) into q' through its entry
    pdf, final ``(1-rho) P(end|q)``), so every loop state is stochastic.
    """
    V = num_phones
    start = np.full(V, smoothing)
    trans = np.full((V, V), smoothing)
    end = np.full(V, smoothing)
    for phones in corpus:
        start[phones[0]] += 1.0
        for a, b in zip(phones[:-1], phones[1:]):
            trans[a, b] += 1.0
        end[phones[-1]] += 1.0
    start /= start.sum()
    z = trans.sum(axis=1) + end
    trans /= z[:, None]
    end /= z
    rho = self_loop
    arcs = [(0, q + 1, 2 * q, float(start[q])) for q in range(V)]
    for q in range(V):
        arcs.append((q + 1, q + 1, 2 * q + 1, rho))
        arcs += [(q + 1, r + 1, 2 * r, (1.0 - rho) * float(trans[q, r])) for r in range(V)]
    finals = np.zeros(V + 1)
    finals[1:] = (1.0 - rho) * end
    return ChainGraph(arcs, V + 1, 2 * V, 0, finals)


def train(num_phones: int = 6, num_utterances: int = 40, frames_per_phone: int = 8,
          epochs: int = 150, learning_rate: float = 6.0, seed: int = 0, noise: float = 0.2,
          leak: float = 1e-5, device=None) -> TrainResult:
    """Train an affine acoustic model with ChainLoss + autograd on the GPU.

    Deterministic for a fixed seed (the LF-MMI kernels are deterministic).
    """
    import torch

    from .loss import ChainLoss

    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    rng = np.random.default_rng(seed)
    corpus = synthesize_corpus(rng, num_phones, num_utterances)
    targets = [expand_alignment(p, frames_per_phone, rng) for p in corpus]
    D = 2 * num_phones
    lengths = np.asarray([len(t) for t in targets], dtype=np.int64)
    T = int(lengths.max())
    feats = np.zeros((len(corpus), T, D), dtype=np.float32)
    for b, tgt in enumerate(targets):
        x = noise * rng.standard_normal((len(tgt), D))
        x[np.arange(len(tgt)), tgt] += 1.0
        feats[b, :len(tgt)] = x
    nums = [numerator_graph(p, num_phones) for p in corpus]   # caller order, any lengths
    criterion = ChainLoss(bigram_denominator(corpus, num_phones),
                          FBOptions(leak_coefficient=leak), normalize_by_frames=True)

    x = torch.tensor(feats, device=dev)
    lens = torch.tensor(lengths, dtype=torch.int32, device=dev)
    model = torch.nn.Linear(D, D).to(dev)
    with torch.no_grad():
        model.weight.zero_()
        model.bias.zero_()
    opt = torch.optim.SGD(model.parameters(), lr=learning_rate)
    res = TrainResult(total_frames=int(lengths.sum()))
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(epochs):
        opt.zero_grad(set_to_none=True)
        loss = criterion(model(x), lens, nums)
        loss.backward()
        opt.step()
        res.losses.append(float(loss.detach()))
    torch.cuda.synchronize(dev)
    res.frames_per_s = res.total_frames * epochs / (time.perf_counter() - t0)
    with torch.no_grad():
        pred = model(x).argmax(dim=-1).cpu().numpy()
    correct = sum(int((pred[b, :len(t)] == t).sum()) for b, t in enumerate(targets))
    res.accuracy = correct / res.total_frames
    return res
