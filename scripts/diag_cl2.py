import sys, os
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2005_09824_b200 as P
from paper_2005_09824_b200 import synth, _backend
from paper_2005_09824_b200.forward_backward import _WORKSPACE
from oracle import oracle as O
w = synth.make_workload("wsj_mono", seed=3, batch_size=8)
batch, nums, den = w.build(P)
ref = O.chain_loss(batch, nums, den, leak=1e-5)
for serial in (False, True):
    if serial: os.environ["LFMMI_SERIAL_CHAIN"] = "1"
    for rep in range(3):
        res = P.chain_loss(batch, nums, den)
        d = np.abs(res.grad - ref.grad)
        print("serial", serial, "rep", rep, "grad err", d.max(), "bad items", sorted(set(int(b) for b in np.argwhere(d > 1e-4)[:, 0])))
# inspect gamma_num in the workspace after a concurrent call
os.environ.pop("LFMMI_SERIAL_CHAIN")
ext = _backend.ext()
res = P.chain_loss(batch, nums, den)
ws = list(_WORKSPACE.values())[0]
ng = P.device_graphs(nums); dg = P.device_graphs(den)
B, T, D = batch.values.shape
nb = ws.numel()
es = 4
gam_b = B * T * D * es
per_frame = (((1000 + 3)//4*4) + ((nums.max_states + 3)//4*4)) * es
cap = (nb - gam_b - 1024) // per_frame
al = lambda x: (x + 255) & ~255
den_b = al(((1000+3)//4*4) * cap * es); num_b = al(((nums.max_states+3)//4*4) * cap * es)
gam = ws[den_b + num_b: den_b + num_b + gam_b].view(torch.float32).view(B, T, D).cpu().numpy()
fbn = O.forward_backward(batch, nums, leak=1e-5)
print("gamma_num in workspace err", np.abs(gam - fbn.posteriors).max(), "per item", [float(np.abs(gam[b] - fbn.posteriors[b]).max()) for b in range(B)])
