"""Host cost of one chain_loss_packed call (Python + C++ dispatch, no sync) against
its device step time, per config: is the end-to-end loop host-bound?

    python scripts/host_overhead.py hmm wsj_mono
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2005_09824_b200 as P  # noqa: E402
from paper_2005_09824_b200 import synth  # noqa: E402

for cfg in sys.argv[1:] or ["hmm", "wsj_mono"]:
    w = synth.make_workload(cfg, seed=0)
    batch, nums, den = w.build(P)
    L = batch.lengths
    tf, tm = int(L.sum()), int(L.max())
    padded = torch.tensor(batch.values, dtype=torch.float32)
    x = torch.cat([padded[b, :int(L[b])] for b in range(len(L))]).cuda()
    l = torch.tensor(L, dtype=torch.int32).cuda()
    g = torch.empty_like(x)

    def call():
        return P.chain_loss_packed(x, l, nums, den, max_frames=tm, total_frames=tf, grad=g)

    for _ in range(5):
        call()
    torch.cuda.synchronize()
    n = 50
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    t0 = time.perf_counter()
    for _ in range(n):
        call()
    host_ms = (time.perf_counter() - t0) / n * 1e3
    e.record()
    torch.cuda.synchronize()
    dev_ms = s.elapsed_time(e) / n
    # split the host time: graph lookups / checks vs the C++ launch call
    t0 = time.perf_counter()
    for _ in range(n):
        P.loss.device_graphs(nums, x.device, linear_ok=True)
        P.loss.device_graphs(P.loss._as_graph_batch(den, len(L)), x.device)
    look_ms = (time.perf_counter() - t0) / n * 1e3
    torch.cuda.synchronize()
    print(f"{cfg}: host {host_ms:.3f} ms/call (graph lookups {look_ms:.3f}), "
          f"back-to-back device {dev_ms:.3f} ms/step", flush=True)
