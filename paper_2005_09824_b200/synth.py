"""Seeded synthetic LF-MMI workloads.

Reproduces the survey's calibration recipe draw-for-draw with
``np.random.default_rng(seed)``: denominator (ring backbone + random arcs,
sparse finals, near-stochastic normalisation), then lengths, then
log-likelihoods ~ N(0, 2), then per-utterance linear numerators over a
``D // 2``-phone topology (the reference's ``build_numerator`` with its
default ``PhoneTopology``: entry prob 1, self-loop 0.5, advance 0.5, final
0.5 — toy_builder.py:218-265).  Probabilities and log-likelihoods are rounded
to fp32 so that the fp64 reference and the fp32 kernels see identical inputs.

``Workload.build(lib)`` instantiates the graphs and batch with any module
exposing the reference API (this package, or ``chainloss`` itself for the
CPU baseline), so both sides consume byte-identical inputs.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = ["CONFIGS", "Workload", "make_workload", "numerator_arcs"]

# name: (S, I, D, B, T_lo, T_hi)   — BASELINE.json configs 1-5
# plus "hmm": a phone-bigram denominator shaped like the reference's own
# build_denominator (toy_builder.py:268-310) — 42 phones, S = 43, I = 1848, D = 84,
# ~2 distinct pdfs per destination — with LM-weighted numerators.
CONFIGS = {
    "hmm": (43, 1848, 84, 128, 150, 300),
    "toy": (50, 200, 10, 4, 25, 50),
    "wsj_mono": (1000, 10000, 84, 128, 150, 300),
    "wsj_biphone": (3000, 30000, 2000, 128, 250, 500),
    "large": (20000, 200000, 2000, 64, 250, 500),
    "sweep": (1000, 10000, 84, 1024, 50, 1500),
}


def den_arcs(rng: np.random.Generator, S: int, I: int, D: int, fp32: bool = True):
    """Denominator arcs and finals, Appendix B draw order."""
    ring_pdf = np.empty(S, dtype=np.int64)
    ring_p = np.empty(S, dtype=np.float64)
    for s in range(S):  # scalar draws, interleaved, as in the recipe
        ring_pdf[s] = int(rng.integers(0, D))
        ring_p[s] = float(rng.uniform(0.2, 1.2))
    k = I - S
    fr = rng.integers(0, S, k)
    to = rng.integers(0, S, k)
    pd = rng.integers(0, D, k)
    pr = rng.uniform(0.2, 1.2, k)
    finals = np.zeros(S)
    sel = rng.random(S) < 0.1
    finals[sel] = rng.uniform(0.2, 1.0, sel.sum())
    finals[S - 1] = 0.5
    src = np.concatenate([np.arange(S), fr]).astype(np.int64)
    dst = np.concatenate([(np.arange(S) + 1) % S, to]).astype(np.int64)
    pdf = np.concatenate([ring_pdf, pd]).astype(np.int64)
    prob = np.concatenate([ring_p, pr])
    out = np.bincount(src, weights=prob, minlength=S)
    prob = prob / (out[src] + finals[src])
    if fp32:
        prob = prob.astype(np.float32).astype(np.float64)
        finals = finals.astype(np.float32).astype(np.float64)
    return src, dst, pdf, prob, finals


def bigram_lm(rng: np.random.Generator, num_phones: int):
    """Random bigram phone LM (begin / transition / end probabilities), the
    quantities the reference's BigramLM holds (toy_builder.py:67-100)."""
    start = rng.random(num_phones) + 0.05
    trans = rng.random((num_phones, num_phones)) ** 2 + 0.01
    end = rng.random(num_phones) * 0.3 + 0.05
    start /= start.sum()
    norm = trans.sum(axis=1) + end
    return start, trans / norm[:, None], end / norm


def hmm_den_arcs(rng: np.random.Generator, num_phones: int, self_loop: float = 0.5,
                 fp32: bool = True):
    """Phone-bigram denominator in the shape of build_denominator
    (toy_builder.py:268-310): state 0 enters every phone's loop state j + 1
    through its entry pdf 2j with P(j | begin); loop state j + 1 self-loops on
    pdf 2j + 1 with the topology weight and hands (1 - rho) P(k | j) to every
    phone k through its entry pdf; final (1 - rho) P(end | j).  Returns the
    arcs, finals and the LM (for LM-weighted numerators)."""
    lm = bigram_lm(rng, num_phones)
    start, trans, end = lm
    P = num_phones
    src = [np.zeros(P, dtype=np.int64), np.arange(1, P + 1)]
    dst = [np.arange(1, P + 1), np.arange(1, P + 1)]
    pdf = [2 * np.arange(P), 2 * np.arange(P) + 1]
    prob = [start, np.full(P, self_loop)]
    j, k = np.meshgrid(np.arange(P), np.arange(P), indexing="ij")
    src.append(j.ravel() + 1)
    dst.append(k.ravel() + 1)
    pdf.append(2 * k.ravel())
    prob.append((1.0 - self_loop) * trans.ravel())
    src, dst, pdf, prob = (np.concatenate(x) for x in (src, dst, pdf, prob))
    finals = np.zeros(P + 1)
    finals[1:] = (1.0 - self_loop) * end
    if fp32:
        prob = prob.astype(np.float32).astype(np.float64)
        finals = finals.astype(np.float32).astype(np.float64)
    return (src.astype(np.int64), dst.astype(np.int64), pdf.astype(np.int64), prob, finals), lm


def numerator_arcs(phones, num_phones: int, self_loop: float = 0.5, lm=None):
    """Linear numerator of a phone sequence (toy_builder.py:218-265, lm=None)."""
    n = len(phones)
    f32 = lambda x: float(np.float32(x))  # noqa: E731
    if lm is None:
        entry, advance, final = 1.0, [1.0 - self_loop] * (n - 1), 1.0 - self_loop
    else:  # build_numerator(phones, topo, lm): weights of the matching den paths
        start, trans, end = lm
        entry = f32(start[phones[0]])
        advance = [f32((1.0 - self_loop) * trans[a, b]) for a, b in zip(phones, phones[1:])]
        final = f32((1.0 - self_loop) * end[phones[-1]])
    arcs = [(0, 1, 2 * int(phones[0]), entry)]
    for k, p in enumerate(phones):
        arcs.append((k + 1, k + 1, 2 * int(p) + 1, self_loop))
        if k + 1 < n:
            arcs.append((k + 1, k + 2, 2 * int(phones[k + 1]), advance[k]))
    finals = np.zeros(n + 1)
    finals[n] = final
    return arcs, n + 1, finals


@dataclass
class Workload:
    name: str
    seed: int
    S: int
    I: int
    D: int
    lengths: np.ndarray                 # input order
    seqs: list                          # (T_b, D) float64 (fp32-exact)
    den: tuple                          # (src, dst, pdf, prob, finals)
    num_phones: list = field(default_factory=list)
    lm: tuple | None = None  # "hmm": numerators weighted by the den's LM

    @property
    def total_frames(self) -> int:
        return int(np.sum(self.lengths))

    def den_graph(self, lib):
        src, dst, pdf, prob, finals = self.den
        arcs = list(zip(src.tolist(), dst.tolist(), pdf.tolist(), prob.tolist()))
        return lib.ChainGraph(arcs, self.S, self.D, 0, finals)

    def build(self, lib, den_graph=None):
        """(batch, numerators, denominator) with ``lib``'s classes, sorted order."""
        batch = lib.make_batch(self.seqs)
        den = den_graph if den_graph is not None else self.den_graph(lib)
        nums = []
        for phones in self.num_phones:
            arcs, n, finals = numerator_arcs(phones, self.D // 2, lm=self.lm)
            nums.append(lib.ChainGraph(arcs, n, self.D, 0, finals))
        nums = [nums[i] for i in batch.order_map]
        return batch, lib.ChainGraphBatch.from_graphs(nums), lib.ChainGraphBatch.broadcast(
            den, len(self.seqs))


def make_workload(name: str = "wsj_mono", seed: int = 0, batch_size: int | None = None,
                  fp32: bool = True) -> Workload:
    """Draw a workload for one of :data:`CONFIGS` (optionally overriding B)."""
    S, I, D, B, t_lo, t_hi = CONFIGS[name]
    if batch_size is not None:
        B = int(batch_size)
    rng = np.random.default_rng(seed)
    lm = None
    if name == "hmm":
        den, lm = hmm_den_arcs(rng, D // 2, fp32=fp32)
    else:
        den = den_arcs(rng, S, I, D, fp32)
    lengths = rng.integers(t_lo, t_hi + 1, B)
    seqs = []
    for t in lengths:
        x = rng.normal(0.0, 2.0, size=(int(t), D))
        if fp32:
            x = x.astype(np.float32).astype(np.float64)
        seqs.append(x)
    num_phones = [rng.integers(0, D // 2, max(1, int(t) // 3)).tolist() for t in lengths]
    return Workload(name, seed, S, I, D, np.asarray(lengths, dtype=np.int64), seqs, den,
                    num_phones, lm)
