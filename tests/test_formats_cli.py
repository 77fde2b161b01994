"""Text-FST / PCTN formats and the CLI front-end.

Fixtures in tests/golden/cli were produced by the REAL reference
(tests/golden/make_cli_golden.py): its make-num / make-den graphs, seeded
logits, and the stdout / gradient file of its own `loss` and `grad` commands.
"""

import contextlib
import io
import math
import os
import re

import numpy as np
import pytest

import paper_2005_09824_b200 as P
from paper_2005_09824_b200 import cli, formats, synth

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cli")
D = 6


def _fsts():
    names = sorted(os.listdir(os.path.join(GOLD, "nums")))
    return [(n.replace(".fst", ""), os.path.join(GOLD, "nums", n)) for n in names] + [
        ("den", os.path.join(GOLD, "den.fst"))]


@pytest.mark.parametrize("key,path", _fsts())
def test_native_parse_matches_reference(key, path):
    ref = np.load(os.path.join(GOLD, "parsed.npz"))
    g = formats.parse_fst_text(open(path).read(), D)
    for attr in ("forward_from", "forward_to", "forward_pdf", "forward_probs", "final_probs"):
        np.testing.assert_array_equal(np.asarray(getattr(g, attr)), ref[f"{key}/{attr}"])
    assert formats.serialize_fst_text(g) == str(ref[f"{key}/serialized"])


def test_serialize_round_trip_is_exact():
    """States are re-indexed by first appearance (fst_io.py:12-17): the first
    round trip relabels; weights are printed with 17 digits, so probabilities
    come back to within an ulp (exp(-(-log p)))."""
    w = synth.make_workload("toy", seed=2, batch_size=2)
    src, dst, pdf, prob, finals = w.den
    g = P.ChainGraph(list(zip(src.tolist(), dst.tolist(), pdf.tolist(), prob.tolist())), w.S,
                     w.D, 0, finals)
    t1 = formats.serialize_fst_text(g)
    g2 = formats.parse_fst_text(t1, w.D)
    assert (g2.num_states, g2.num_transitions) == (g.num_states, g.num_transitions)
    np.testing.assert_allclose(np.sort(g2.forward_probs), np.sort(g.forward_probs), rtol=1e-15)
    np.testing.assert_allclose(np.sort(g2.final_probs), np.sort(g.final_probs), rtol=1e-15)
    # the relabelling is first appearance in the text: rebuild it and compare arcs
    relabel = {}
    for line in t1.splitlines():
        for tok in line.split()[: 2 if len(line.split()) >= 3 else 1]:
            relabel.setdefault(int(tok), len(relabel))
    mapped = sorted((relabel[a], relabel[b], c, p) for a, b, c, p in zip(
        g.forward_from.tolist(), g.forward_to.tolist(), g.forward_pdf.tolist(),
        g.forward_probs.tolist()))
    got = sorted(zip(g2.forward_from.tolist(), g2.forward_to.tolist(), g2.forward_pdf.tolist(),
                     g2.forward_probs.tolist()))
    assert [m[:3] for m in mapped] == [x[:3] for x in got]
    np.testing.assert_allclose([x[3] for x in got], [m[3] for m in mapped], rtol=1e-15)


@pytest.mark.parametrize("text,match", [
    ("0 1 0 0.5\n1 0\n", "line 1: label 0 is reserved"),
    ("0 1 9\n1\n", "line 1: label 9 exceeds num_pdfs=6"),
    ("# c\n0 x 1\n1\n", "line 2: dst state is not an integer"),
    ("0 1 1 abc\n1\n", "line 1: weight is not a number"),
    ("0 1 1 inf\n1\n", "line 1: weight must be finite"),
    ("0 1 1\n1\n1 0.5\n", "line 3: duplicate final line"),
    ("0 1 1\n", "no final state"),
    ("\n# only comments\n", "empty FST"),
    ("0 1 1 0 7\n1\n", "line 1: expected 1-2 \\(final\\) or 3-4 \\(arc\\) fields, got 5"),
    ("0 -1 1\n1\n", "line 1: dst state must be non-negative"),
])
def test_parse_errors_carry_line_numbers(text, match):
    with pytest.raises(formats.FstParseError, match=match):
        formats.parse_fst_text(text, D)


def test_pctn_round_trip_and_errors(tmp_path):
    rng = np.random.default_rng(0)
    for shape in [(), (3,), (2, 3), (2, 3, 4), (1, 2, 3, 2)]:
        a = rng.normal(size=shape)
        formats.write_array(tmp_path / "a.pctn", a)
        b = formats.read_array(tmp_path / "a.pctn")
        assert b.shape == a.shape and b.tobytes() == np.asarray(a, np.float64).tobytes()
    ref = formats.read_array(os.path.join(GOLD, "logits.pctn"))
    assert ref.shape == (3, 12, D)
    raw = (tmp_path / "a.pctn").read_bytes()
    for bad, match in [(raw[:10], "truncated header"), (b"XXXX" + raw[4:], "bad magic"),
                       (raw + b"\0", "trailing bytes"), (raw[:-8], "truncated payload")]:
        (tmp_path / "b.pctn").write_bytes(bad)
        with pytest.raises(ValueError, match=match):
            formats.read_array(tmp_path / "b.pctn")
    with pytest.raises(ValueError, match="at most 4"):
        formats.write_array(tmp_path / "c.pctn", np.zeros((1,) * 5))


def _run(argv):
    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        code = cli.main(argv)
    return code, out.getvalue(), err.getvalue()


def _common():
    return ["--logits", os.path.join(GOLD, "logits.pctn"), "--lengths",
            os.path.join(GOLD, "lengths.txt"), "--num-fsts", os.path.join(GOLD, "nums"),
            "--den-fst", os.path.join(GOLD, "den.fst")]


def test_cli_usage_errors_exit_one(tmp_path):
    code, _, err = _run(["loss", "--logits", str(tmp_path / "nope.pctn"), "--num-fsts", "x",
                         "--den-fst", "y"])
    assert code == 1 and "nope.pctn" in err
    code, _, err = _run(["frobnicate"])
    assert code == 1
    (tmp_path / "bad.txt").write_text("9\n7\n13\n")
    args = _common()
    args[3] = str(tmp_path / "bad.txt")
    code, _, err = _run(["loss", *args])
    assert code == 1 and "not in [1, 12]" in err


def _numbers(text):
    utt = [tuple(float(x) for x in m) for m in re.findall(
        r"num=([-\d.]+) den=([-\d.]+) F=([-\d.]+)", text)]
    batch = re.search(r"batch: F=([-\d.]+) loss=([-\d.]+) frames=(\d+) failed=(\d+)", text)
    return utt, tuple(float(x) for x in batch.groups())


@pytest.mark.gpu
@pytest.mark.parametrize("precision,tol", [("fp64", 1e-9), ("fp32", 1e-5)])
def test_cli_loss_and_grad_match_reference(cuda, tmp_path, precision, tol):
    code, out, _ = _run(["loss", *_common(), "--per-frame", "--precision", precision])
    ref = open(os.path.join(GOLD, "loss.out")).read()
    assert code == 0 and ref.startswith("exit=0")
    (u, b), (ru, rb) = _numbers(out), _numbers(ref)
    assert len(u) == len(ru) == 3 and b[2:] == rb[2:]
    for x, y in zip([v for t in u for v in t] + list(b[:2]), [v for t in ru for v in t] + list(rb[:2])):
        assert abs(x - y) <= tol * max(1.0, abs(y)) + 1e-9, (x, y)
    code, out, _ = _run(["grad", *_common(), "--out", str(tmp_path / "g.pctn"),
                         "--precision", precision])
    assert code == 0 and "wrote" in out
    g = formats.read_array(tmp_path / "g.pctn")
    gr = formats.read_array(os.path.join(GOLD, "grad.pctn"))
    assert g.shape == gr.shape
    assert np.abs(g - gr).max() <= (1e-9 if precision == "fp64" else 1e-4)


@pytest.mark.gpu
def test_cli_identical_graphs_zero_objective(cuda, tmp_path):
    (tmp_path / "g.fst").write_text("0 0 1 0\n0 0\n")
    formats.write_array(tmp_path / "l.pctn", np.zeros((1, 4, 1)))
    code, out, _ = _run(["loss", "--logits", str(tmp_path / "l.pctn"), "--num-fsts",
                         str(tmp_path / "g.fst"), "--den-fst", str(tmp_path / "g.fst")])
    assert code == 0
    assert abs(float(re.search(r"batch: F=([-\d.]+)", out).group(1))) < 1e-10


@pytest.mark.gpu
def test_cli_train_demo(cuda):
    code, out, _ = _run(["train-demo", "--epochs", "40", "--utterances", "12"])
    assert code == 0 and "accuracy=" in out
    acc = float(re.search(r"accuracy=([\d.]+)", out).group(1))
    assert math.isfinite(acc)
