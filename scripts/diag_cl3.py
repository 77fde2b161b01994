import sys, os
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2005_09824_b200 as P
from paper_2005_09824_b200 import synth, _backend
from oracle import oracle as O
ext = _backend.ext()
w = synth.make_workload("wsj_mono", seed=3, batch_size=8)
batch, nums, den = w.build(P)
ref = O.chain_loss(batch, nums, den, leak=1e-5)
dev = torch.device("cuda", 0)
values = torch.tensor(batch.values, dtype=torch.float32, device=dev)
lengths = torch.tensor(batch.lengths, dtype=torch.int32, device=dev)
ng = P.device_graphs(nums, dev); dg = P.device_graphs(den, dev)
B, T, D = values.shape
nbytes = ext.chain_loss_workspace_size(ng.handle, dg.handle, B, T, D, int(batch.lengths.sum()), 0)
print("nbytes", nbytes)
def run(ws, tag):
    grad = torch.empty_like(values)
    f64 = dict(dtype=torch.float64, device=dev); i32 = dict(dtype=torch.int32, device=dev)
    nl, dl = torch.empty(B, **f64), torch.empty(B, **f64)
    nf, df = torch.empty(B, **i32), torch.empty(B, **i32)
    tot = torch.empty(3, **f64)
    ext.chain_loss(ng.handle, ng.row_map, dg.handle, dg.row_map, values, lengths, 1e-5, 1e-300, None, None, ws, grad, nl, dl, nf, df, tot)
    torch.cuda.synchronize()
    d = np.abs(grad.double().cpu().numpy() - ref.grad)
    print(tag, "err", d.max(), "bad", sorted(set(int(b) for b in np.argwhere(d > 1e-4)[:, 0])), "fails", nf.cpu().tolist(), df.cpu().tolist())
ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
for i in range(3): run(ws, f"exact-size ws rep{i}")
for i in range(2):
    ws.zero_(); run(ws, f"zeroed ws rep{i}")
for i in range(2):
    ws.view(torch.float32)[: nbytes // 4].fill_(float('nan')); run(ws, f"nan ws rep{i}")
big = torch.empty(nbytes * 3, dtype=torch.uint8, device=dev)
for i in range(2): run(big, f"big ws rep{i}")
