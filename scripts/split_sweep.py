"""Debug: den pass time of the split kernel vs cluster count (WSJ-mono)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2005_09824_b200 as P
from paper_2005_09824_b200 import synth

cfg = sys.argv[1] if len(sys.argv) > 1 else "wsj_mono"
w = synth.make_workload(cfg, seed=0)
batch, nums, den = w.build(P)
v = torch.tensor(batch.values, dtype=torch.float32, device="cuda")
l = torch.tensor(batch.lengths, dtype=torch.int32, device="cuda")
g = torch.empty_like(v)
tf = int(batch.lengths.sum())
def timeit(fn, n=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n
den_alone = lambda: P.forward_backward_device(v, l, den, posteriors=g, mode=3, total_frames=tf)
step = lambda: P.chain_loss_device(v, l, nums, den, total_frames=tf, grad=g)
os.environ["LFMMI_SPLIT"] = "0"
print(cfg, "tile den", round(timeit(den_alone), 3), "step", round(timeit(step), 3), flush=True)
os.environ["LFMMI_SPLIT"] = "1"
for nc in sys.argv[2:] if len(sys.argv) > 2 else ["16", "32", "48", "56", "60", "64", "74"]:
    os.environ["LFMMI_SPLIT_CLUSTERS"] = nc
    print(cfg, "split clusters", nc, "den", round(timeit(den_alone), 3), "step", round(timeit(step), 3), flush=True)
