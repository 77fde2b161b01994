"""Generate CLI / format golden fixtures with the REAL reference (run in the
build container, where /root/reference exists; the outputs are committed).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_cli_golden.py

Writes tests/golden/cli/: phones.txt, corpus.txt, nums/*.fst, den.fst (from the
reference's make-num / make-den), logits.pctn + lengths.txt (seeded), the
reference's `loss` / `grad` stdout (loss.out, grad.out), grad.pctn, and
parsed.npz (the reference parse of every FST: arrays of the ChainGraph).
"""
import contextlib
import io
import os
import sys

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_lfmmi")
sys.dont_write_bytecode = True
REF_SRC = os.environ.get("CHAINLOSS_REF_SRC", "/root/reference/pkg/src")
if REF_SRC not in sys.path:
    sys.path.insert(0, REF_SRC)
import chainloss as C  # noqa: E402
from chainloss.cli import main  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cli")


def run(argv):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        code = main(argv)
    return code, buf.getvalue()


def main_():
    os.makedirs(OUT, exist_ok=True)
    p = lambda *a: os.path.join(OUT, *a)  # noqa: E731
    open(p("phones.txt"), "w").write("aa\nbb\ncc\n")
    open(p("corpus.txt"), "w").write("aa bb | cc\nbb cc\ncc aa aa\n")
    assert main(["make-num", "--corpus", p("corpus.txt"), "--phones", p("phones.txt"),
                 "--out-dir", p("nums")]) == 0
    assert main(["make-den", "--corpus", p("corpus.txt"), "--phones", p("phones.txt"),
                 "--out", p("den.fst")]) == 0
    rng = np.random.default_rng(7)
    D, lengths = 6, [9, 7, 12]
    values = np.zeros((3, 12, D))
    for b, n in enumerate(lengths):
        values[b, :n] = rng.normal(0, 1, (n, D)).astype(np.float32)  # fp32-exact inputs
    C.write_array(p("logits.pctn"), values)
    open(p("lengths.txt"), "w").write("".join(f"{n}\n" for n in lengths))
    common = ["--logits", p("logits.pctn"), "--lengths", p("lengths.txt"),
              "--num-fsts", p("nums"), "--den-fst", p("den.fst")]
    code, out = run(["loss", *common, "--per-frame"])
    open(p("loss.out"), "w").write(f"exit={code}\n" + out.replace(OUT, "<dir>"))
    code, out = run(["grad", *common, "--out", p("grad.pctn")])
    open(p("grad.out"), "w").write(f"exit={code}\n" + out.replace(OUT, "<dir>"))
    parsed = {}
    files = sorted(os.listdir(p("nums"))) 
    for name in files + ["den.fst"]:
        path = p("nums", name) if name != "den.fst" else p("den.fst")
        g = C.parse_fst_text(open(path).read(), D)
        key = name.replace(".fst", "")
        for attr in ("forward_from", "forward_to", "forward_pdf", "forward_probs", "final_probs"):
            parsed[f"{key}/{attr}"] = np.asarray(getattr(g, attr))
        parsed[f"{key}/serialized"] = np.array(C.serialize_fst_text(g))
    np.savez(p("parsed.npz"), **parsed)
    print("wrote", OUT)


if __name__ == "__main__":
    main_()
