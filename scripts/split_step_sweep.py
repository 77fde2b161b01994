"""A/B: two-pass WSJ-mono step time vs split-kernel cluster count and midpoint (env overrides)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2005_09824_b200 as P
from paper_2005_09824_b200 import synth

w = synth.make_workload("wsj_mono", seed=0)
batch, nums, den = w.build(P)
v = torch.tensor(batch.values, dtype=torch.float32, device="cuda")
l = torch.tensor(batch.lengths, dtype=torch.int32, device="cuda")
g = torch.empty_like(v)
tf = int(batch.lengths.sum())
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def timeit(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(n):
        flush.fill_(1)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        tot += s.elapsed_time(e)
    return tot / n


step = lambda: P.chain_loss_device(v, l, nums, den, total_frames=tf, grad=g)
for rep in range(2):
    for nc in ["62", "63", "64", "65", "66"]:
        for h in ["32", "33", "34"]:
            P._backend.ext().set_option("split_clusters", nc)
            P._backend.ext().set_option("split_h64", h)
            print("rep", rep, "clusters", nc, "h64", h, "step_ms", round(timeit(step), 4), flush=True)
