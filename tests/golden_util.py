"""Load tests/golden/*.npz (recorded from the reference by make_golden.py)
into this package's drop-in classes."""

import glob
import os

import numpy as np

import paper_2005_09824_b200 as P

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def names(prefix=""):
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, prefix + "*.npz")))


def _graph(z, prefix):
    arcs = z[f"{prefix}_arcs"]
    S, D, init = (int(v) for v in z[f"{prefix}_meta"])
    tr = [(int(a), int(b), int(c), float(p)) for a, b, c, p in arcs]
    g = P.ChainGraph(tr, S, D, init, z[f"{prefix}_finals"])
    # Adopt the reference's backward_* order (its summation order) verbatim.
    bw = z[f"{prefix}_bw_arcs"]
    if len(bw):
        g.backward_from = bw[:, 0].astype(np.uint32)
        g.backward_to = bw[:, 1].astype(np.uint32)
        g.backward_pdf = bw[:, 2].astype(np.uint32)
        g.backward_probs = bw[:, 3].copy()
    return g


def load(name):
    z = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    batch = P.LogLikBatch(z["values"], z["lengths"], z["valid_batch_sizes"], z["order_map"])
    nums = P.ChainGraphBatch.from_graphs([_graph(z, f"num{k}") for k in range(int(z["num_graphs"]))])
    den = P.ChainGraphBatch.broadcast(_graph(z, "den"), batch.batch_size)
    return batch, nums, den, float(z["leak"]), z
