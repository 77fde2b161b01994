"""Dump the WSJ-mono denominator (seed 0) for scripts/sched/eval_schedule.cpp."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2005_09824_b200 import synth

w = synth.make_workload("wsj_mono", seed=0, batch_size=2)
src, dst, pdf, prob, fin = w.den
os.makedirs("/tmp/sched", exist_ok=True)
with open("/tmp/sched/den.bin", "wb") as f:
    np.array([w.S, w.D, len(src)], np.int32).tofile(f)
    for a in (src, dst, pdf):
        a.astype(np.int32).tofile(f)
    prob.astype(np.float64).tofile(f)
