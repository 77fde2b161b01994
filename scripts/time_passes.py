"""Debug: den / num pass times alone and the chain step, for one config."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2005_09824_b200 as P
from paper_2005_09824_b200 import synth

cfg = sys.argv[1] if len(sys.argv) > 1 else "sweep"
w = synth.make_workload(cfg, seed=0)
batch, nums, den = w.build(P)
v = torch.tensor(batch.values, dtype=torch.float32, device="cuda")
l = torch.tensor(batch.lengths, dtype=torch.int32, device="cuda")
g = torch.empty_like(v)
tf = int(batch.lengths.sum())
def timeit(fn, n=3):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n
def env(**kw):
    for k in ("LFMMI_TILE_SINGLE_X", "LFMMI_NO_NUM_ROOM"):
        os.environ.pop(k, None)
    os.environ.update(kw)
den_alone = lambda: P.forward_backward_device(v, l, den, posteriors=g, mode=3, total_frames=tf)
num_alone = lambda: P.forward_backward_device(v, l, nums, posteriors=g, mode=0, total_frames=tf)
step = lambda: P.chain_loss_device(v, l, nums, den, total_frames=tf, grad=g)
for label, kw in (("xdb", {}), ("single-x", {"LFMMI_TILE_SINGLE_X": "1"})):
    env(**kw); print(cfg, "den alone", label, round(timeit(den_alone), 3), "ms", flush=True)
env(); print(cfg, "num alone", round(timeit(num_alone), 3), "ms", flush=True)
env(); print(cfg, "step (room for num)", round(timeit(step), 3), "ms", flush=True)
env(LFMMI_NO_NUM_ROOM="1"); print(cfg, "step (no room)", round(timeit(step), 3), "ms", flush=True)
env(); print(cfg, "den alone xdb again", round(timeit(den_alone), 3), "ms", flush=True)
