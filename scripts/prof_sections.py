"""Debug: per-section cycle breakdown of the fused chain kernel (LFMMI_PROFILE=1)."""
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
P.chain_loss_device(v, l, nums, den, total_frames=int(batch.lengths.sum()))
torch.cuda.synchronize()
os.environ["LFMMI_PROFILE"] = "1"
P.chain_loss_device(v, l, nums, den, total_frames=int(batch.lengths.sum()))
torch.cuda.synchronize()
