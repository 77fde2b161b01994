#!/usr/bin/env python
"""One small LF-MMI loss for compute-sanitizer (tests/test_sanitizers.py).

    compute-sanitizer --tool racecheck python scripts/sanitize_case.py split

Cases pick the kernel under test with the library options (lfmmi_set_option):
  split    denominator fb_split_kernel (2-CTA cluster, DSMEM-free handoff via HBM + cluster barrier)
  tile     denominator fb_tile_kernel<512> with double-buffered posterior slots (XDB)
  tile1x   ... single slot buffer
  stream2  large-graph fb_stream_kernel<1024,2> (2-CTA cluster, DSMEM exchange)
  stream1  fb_stream_kernel<1024,1> reading slot rows straight from L2
  ring     fb_stream_kernel<1024,1> with its TMA slot ring (cp.async.bulk + mbarrier)
  ssplit   fb_streamsplit_kernel (forward | backward clusters, DSMEM scalars, kappa recursion)
           with its TMA slot ring; ssplit0 the same reading slot rows from L2
  lin16    numerators with S > 256 on the two-warps-per-direction linear kernel (one 900-frame
           utterance; racecheck over the 64-thread exchange barriers)
  tilep    fb_tile_kernel<512> XDB as 2 persistent CTAs (in-kernel LPT, utterances back to back)
  hmm      phone-bigram den on fb_split_kernel with 8 lanes per state (xor-shuffle sums)
  numtile  numerators on the generic fb_tile_kernel<128> (linear kernel disabled)
every case also runs the linear-chain numerator kernel (except numtile) and
the combine kernel.  Utterances are short (<= 24 frames) to keep the
instrumented run within minutes; the result is checked against the oracle.
"""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2005_09824_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2005_09824_b200 import _backend, synth  # noqa: E402

CASES = {
    "split": ("wsj_mono", 3, dict(split=1, split_clusters=2)),
    "tile": ("wsj_mono", 3, dict(split=0)),
    "tile1x": ("wsj_mono", 3, dict(split=0, tile_xdb=0)),
    "stream2": ("wsj_biphone", 2, dict(stream_mode="1024x2")),
    "stream1": ("wsj_biphone", 2, dict(stream_mode="1024x1", stream_ring=0)),
    "ring": ("wsj_biphone", 2, dict(stream_mode="1024x1", stream_ring=1)),
    "ssplit": ("wsj_biphone", 3, dict(stream_mode="split", ssplit_ring=1)),
    "ssplit0": ("wsj_biphone", 3, dict(stream_mode="split")),
    "hmm": ("hmm", 3, dict()),
    "tilep": ("wsj_mono", 3, dict(split=0, tile_persist=2)),
    "lin16": ("wsj_mono", 2, dict()),
    "numtile": ("wsj_mono", 3, dict(linear=0)),
}


def main(case):
    import torch

    config, B, opts = CASES[case]
    ext = _backend.require_cuda()
    for k, v in opts.items():
        ext.set_option(k, str(v))
    w = synth.make_workload(config, seed=2, batch_size=B)
    rng = np.random.default_rng(1)
    T = [24, 17, 9][:B] if case != "lin16" else [900, 12]
    w.seqs = [s[:t] for s, t in zip(w.seqs, T)]
    w.lengths = np.asarray(T, dtype=np.int64)
    w.num_phones = [rng.integers(0, w.D // 2, max(1, t // 3)).tolist() for t in T]
    batch, nums, den = w.build(P)
    res = P.chain_loss(batch, nums, den)
    torch.cuda.synchronize()
    ref = O.chain_loss(batch, nums, den, leak=1e-5)
    err = float(np.abs(res.grad - ref.grad).max())
    rel = abs(res.objective - ref.objective) / max(1.0, abs(ref.objective))
    print(f"case {case}: den kernel {ext.last_den_kernel()}, grad err {err:.2e}, objf rel {rel:.2e}")
    assert err <= 1e-4 and rel <= 1e-5


if __name__ == "__main__":
    main(sys.argv[1])
