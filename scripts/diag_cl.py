import sys, os
sys.path.insert(0, '.')
import numpy as np
import paper_2005_09824_b200 as P
from paper_2005_09824_b200 import synth
from oracle import oracle as O
for B in (8, 128):
    w = synth.make_workload("wsj_mono", seed=3, batch_size=B)
    batch, nums, den = w.build(P)
    ref = O.chain_loss(batch, nums, den, leak=1e-5)
    for rep in range(2):
        res = P.chain_loss(batch, nums, den)
        d = np.abs(res.grad - ref.grad)
        print("B", B, "rep", rep, "obj", res.objective, ref.objective, "grad err", d.max())
        if d.max() > 1e-4:
            items = sorted(set(int(b) for b in np.argwhere(d > 1e-4)[:, 0]))
            print("  bad items", items[:20], len(items))
            b = items[0]
            bt = np.argwhere(d[b] > 1e-4)
            print("  item", b, "T", batch.lengths[b], "bad frames", sorted(set(int(t) for t, _ in bt))[:10], "...", len(bt))
            fbn = P.forward_backward(batch, nums); fbd = P.forward_backward(batch, den)
            g2 = fbn.posteriors - fbd.posteriors
            print("  fb-composed err", np.abs(g2 - ref.grad).max())
            print("  sample", res.grad[b, bt[0][0], :6], ref.grad[b, bt[0][0], :6])
