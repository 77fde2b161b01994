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
CONFIGS = {
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


def numerator_arcs(phones, num_phones: int, self_loop: float = 0.5):
    """Linear numerator of a phone sequence (toy_builder.py:218-265, lm=None)."""
    n = len(phones)
    arcs = [(0, 1, 2 * int(phones[0]), 1.0)]
    for k, p in enumerate(phones):
        arcs.append((k + 1, k + 1, 2 * int(p) + 1, self_loop))
        if k + 1 < n:
            arcs.append((k + 1, k + 2, 2 * int(phones[k + 1]), 1.0 - self_loop))
    finals = np.zeros(n + 1)
    finals[n] = 1.0 - self_loop
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
            arcs, n, finals = numerator_arcs(phones, self.D // 2)
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
                    num_phones)
