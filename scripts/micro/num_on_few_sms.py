"""Experiment: numerator pass time when only (148 - K) SMs are free."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2005_09824_b200 as P
from paper_2005_09824_b200 import synth

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libblocker.so"))
w = synth.make_workload("wsj_mono", seed=0)
batch, nums, den = w.build(P)
v = torch.tensor(batch.values, dtype=torch.float32, device="cuda")
l = torch.tensor(batch.lengths, dtype=torch.int32, device="cuda")
g = torch.empty_like(v)
tf = int(batch.lengths.sum())
sb = torch.cuda.Stream()
num = lambda: P.forward_backward_device(v, l, nums, posteriors=g, mode=0, total_frames=tf)
for _ in range(3): num()
torch.cuda.synchronize()
for K in (0, 100, 120, 128, 136):
    ts = []
    for rep in range(3):
        torch.cuda.synchronize()
        if K:
            lib.launch_blocker(K, int(8e6), ctypes.c_void_p(sb.cuda_stream))  # ~4 ms
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(20000)
        s.record(); num(); e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    print(f"blocked SMs {K:3d}: num pass {min(ts):.3f} ms  {[round(t,3) for t in ts]}", flush=True)
