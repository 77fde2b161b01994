"""Where the e2e leg's fixed cost sits: per-step completion times (events on the
compute stream) and host issue time, packed API, after an L2 flush (as bench.py)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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
hx = [packed.pin_memory() for _ in range(2)]; hl = [lens.pin_memory() for _ in range(2)]
dx = [torch.empty(packed.shape, device="cuda") for _ in range(2)]
dl = [torch.empty(lens.shape, dtype=torch.int32, device="cuda") for _ in range(2)]
g = torch.empty_like(dx[0])
cs, ds = torch.cuda.Stream(), torch.cuda.Stream()
done = [torch.cuda.Event() for _ in range(2)]; used = [torch.cuda.Event() for _ in range(2)]
ht = torch.empty((64, 3), dtype=torch.float64).pin_memory()
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def h2d(i, ev=None):
    j = i & 1
    with torch.cuda.stream(cs):
        cs.wait_event(used[j]); dx[j].copy_(hx[j], non_blocking=True)
        dl[j].copy_(hl[j], non_blocking=True); done[j].record(cs)
        if ev is not None: ev.record(cs)


def run(n, marks=None, host=None):
    h2d(0, marks[0] if marks else None)
    for i in range(n):
        t0 = time.perf_counter()
        if i + 1 < n: h2d(i + 1)
        j = i & 1
        st.wait_event(done[j])
        tot = P.chain_loss_packed(dx[j], dl[j], nums, den, max_frames=tm, total_frames=tf, grad=g)[-1]
        used[j].record(st)
        if marks: marks[i + 1].record(st)
        ds.wait_event(used[j]); tot.record_stream(ds)
        with torch.cuda.stream(ds): ht[i].copy_(tot, non_blocking=True)
        if host is not None: host.append(time.perf_counter() - t0)


for flush_first in (True, False):
    run(3); torch.cuda.synchronize()
    if flush_first:
        flush.fill_(0); torch.cuda.synchronize()
    n = 10
    marks = [E() for _ in range(n + 1)]
    s, e = E(), E()
    host = []
    s.record(cs); run(n, marks, host); e.record(ds); torch.cuda.synchronize()
    print("flush" if flush_first else "noflush", "total_ms", round(s.elapsed_time(e), 3),
          "first_h2d_ms", round(s.elapsed_time(marks[0]), 3),
          "step_done_ms", [round(s.elapsed_time(m), 3) for m in marks[1:]],
          "tail_ms", round(marks[-1].elapsed_time(e), 3),
          "host_us", [round(h * 1e6) for h in host], flush=True)
