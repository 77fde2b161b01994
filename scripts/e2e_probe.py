"""A/B: WSJ-mono step time, padded (B, T, D) vs packed (sum T, D) input, device-resident and
end to end (pinned H2D one step ahead on a copy stream + totals D2H), 10 and 40 steps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2005_09824_b200 as P
from paper_2005_09824_b200 import synth

w = synth.make_workload("wsj_mono", seed=0)
batch, nums, den = w.build(P)
L = batch.lengths
tf, tm = int(L.sum()), int(L.max())
padded = torch.tensor(batch.values, dtype=torch.float32)
packed = torch.cat([padded[b, :int(L[b])] for b in range(len(L))])
lens = torch.tensor(L, dtype=torch.int32)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()


def call(kind, x, l, g):
    if kind == "padded":
        return P.chain_loss_device(x, l, nums, den, total_frames=tf, grad=g)[-1]
    return P.chain_loss_packed(x, l, nums, den, max_frames=tm, total_frames=tf, grad=g)[-1]


for kind, host in (("padded", padded), ("packed", packed)):
    x = host.cuda(); l = lens.cuda(); g = torch.empty_like(x)
    for _ in range(3): call(kind, x, l, g)
    torch.cuda.synchronize()
    t = 0.0
    for _ in range(20):
        flush.fill_(1)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); call(kind, x, l, g); e.record(); torch.cuda.synchronize()
        t += s.elapsed_time(e)
    print(kind, "device step_ms", round(t / 20, 4), "h2d_bytes", host.numel() * 4, flush=True)
    hx = [host.pin_memory() for _ in range(2)]; hl = [lens.pin_memory() for _ in range(2)]
    dx = [torch.empty_like(x) for _ in range(2)]; dl = [torch.empty_like(l) for _ in range(2)]
    cs, ds = torch.cuda.Stream(), torch.cuda.Stream()
    done = [torch.cuda.Event() for _ in range(2)]; used = [torch.cuda.Event() for _ in range(2)]
    ht = torch.empty((64, 3), dtype=torch.float64).pin_memory()

    def h2d(i):
        j = i & 1
        with torch.cuda.stream(cs):
            cs.wait_event(used[j]); dx[j].copy_(hx[j], non_blocking=True)
            dl[j].copy_(hl[j], non_blocking=True); done[j].record(cs)

    def run(n):
        h2d(0)
        for i in range(n):
            if i + 1 < n: h2d(i + 1)
            j = i & 1
            st.wait_event(done[j]); tot = call(kind, dx[j], dl[j], g)
            used[j].record(st); ds.wait_event(used[j]); tot.record_stream(ds)
            with torch.cuda.stream(ds): ht[i].copy_(tot, non_blocking=True)

    for n in (10, 40):
        run(3); torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(cs); run(n); e.record(ds); torch.cuda.synchronize()
        print(kind, "e2e steps", n, "ms_per_step", round(s.elapsed_time(e) / n, 4), flush=True)
