import time, torch, numpy as np, sys
sys.path.insert(0, '.')
import paper_2005_09824_b200 as P
from paper_2005_09824_b200 import synth
for cfg, B in (("wsj_biphone", 8), ("large", 2)):
    t0=time.time()
    w = synth.make_workload(cfg, seed=0, batch_size=B)
    batch, nums, den = w.build(P)
    print(cfg, "build", time.time()-t0, flush=True)
    try:
        t0=time.time(); r = P.chain_loss(batch, nums, den); torch.cuda.synchronize()
        print(cfg, "ok", r.objective, time.time()-t0, flush=True)
    except Exception as e:
        print(cfg, "ERR", repr(e)[:300], flush=True)
