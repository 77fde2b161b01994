import sys, os
sys.path.insert(0, '.')
import numpy as np
import paper_2005_09824_b200 as P
from paper_2005_09824_b200 import synth
from oracle import oracle as O
w = synth.make_workload("wsj_mono", seed=3, batch_size=8)
batch, nums, den = w.build(P)
for prec in ("fp32", "fp64"):
    fb = P.forward_backward(batch, nums, precision=prec)
    ref = O.forward_backward(batch, nums, leak=1e-5)
    d = np.abs(fb.posteriors - ref.posteriors)
    print(prec, "logp err", np.abs(fb.log_probs - ref.log_probs).max(), "post err", d.max())
    bad = np.argwhere(d > 1e-4)
    print(" bad rows (b,t):", sorted(set((int(b), int(t)) for b, t, _ in bad))[:20], "count", len(bad))
    for b in range(batch.batch_size):
        print("  item", b, "T", batch.lengths[b], "S", nums.graph(b).num_states, "maxerr", d[b].max())
