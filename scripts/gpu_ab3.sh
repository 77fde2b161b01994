mkdir -p gpurun_out; : > gpurun_out/ab3.log
one() { env $2 timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('$1', 'ms/step', round(d['ms_per_step'], 4), 'value', round(d['value']/1e6, 3))" >> gpurun_out/ab3.log; }
for r in 1 2; do
one twopass-num32 ""
one twopass-num64 "LFMMI_NUM_GROUP=64"
one twopass-num128 "LFMMI_NUM_GROUP=128"
done
python - >> gpurun_out/ab3.log 2>&1 <<'PY'
import os, sys, torch
sys.path.insert(0, '.')
import paper_2005_09824_b200 as P
from paper_2005_09824_b200 import synth
w = synth.make_workload("wsj_mono", seed=0); batch, nums, den = w.build(P)
v = torch.tensor(batch.values, dtype=torch.float32, device="cuda"); l = torch.tensor(batch.lengths, dtype=torch.int32, device="cuda")
g = torch.empty_like(v)
for grp in ("32", "64", "128"):
    os.environ["LFMMI_NUM_GROUP"] = grp
    for name, gr, mode in (("num", nums, 2), ("den", den, 3)):
        for _ in range(3): P.forward_backward_device(v, l, gr, posteriors=g, mode=mode, total_frames=int(batch.lengths.sum()))
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10): P.forward_backward_device(v, l, gr, posteriors=g, mode=mode, total_frames=int(batch.lengths.sum()))
        e.record(); torch.cuda.synchronize()
        print("alone", name, "group", grp, round(s.elapsed_time(e) / 10, 4), "ms")
PY
