"""Command-line front-end on the GPU backend.

    python -m paper_2005_09824_b200.cli loss  --logits X.pctn[,..] [--lengths F]
                                              --num-fsts DIR|a.fst,.. --den-fst den.fst
                                              [--leak 1e-5] [--per-frame] [--precision fp32|fp64]
    python -m paper_2005_09824_b200.cli grad  ... --out grad.pctn
    python -m paper_2005_09824_b200.cli train-demo [--phones 6 --utterances 40 --epochs 150]

Same inputs, report lines and exit codes as the reference's ``chainloss
loss|grad`` (/root/reference/pkg/src/chainloss/cli.py:1-7, 129-237): 0 on
success, 1 on usage / I/O errors, 2 when an utterance (or all) failed
numerically; the gradient file is in the caller's (unsorted) utterance order.
The reference's graph *builders* (make-num / make-den, toy_builder.py) and the
brute-force gradcheck are graph production / test tooling, out of scope here
(SURVEY.md §2 rows 7-8); train-demo runs this package's torch trainer
(train.py) instead of the reference's numpy one.
"""

from __future__ import annotations

import argparse
import math
import sys
from pathlib import Path

import numpy as np

__all__ = ["main"]


class UsageError(ValueError):
    pass


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # usage errors exit 1, like the reference
        raise UsageError(message)


def _parser():
    p = _Parser(prog="paper_2005_09824_b200.cli", description=__doc__.split("\n")[0])
    sub = p.add_subparsers(dest="command", required=True, parser_class=_Parser)
    for name in ("loss", "grad"):
        q = sub.add_parser(name)
        q.add_argument("--logits", required=True)
        q.add_argument("--lengths")
        q.add_argument("--num-fsts", required=True)
        q.add_argument("--den-fst", required=True)
        q.add_argument("--leak", type=float, default=1e-5)
        q.add_argument("--per-frame", action="store_true")
        q.add_argument("--threads", type=int, help="accepted for compatibility; unused on GPU")
        q.add_argument("--precision", choices=("fp32", "fp64"), default="fp32")
        if name == "grad":
            q.add_argument("--out", required=True)
    d = sub.add_parser("train-demo")
    d.add_argument("--phones", type=int, default=6)
    d.add_argument("--utterances", type=int, default=40)
    d.add_argument("--frames-per-phone", type=int, default=8)
    d.add_argument("--epochs", type=int, default=150)
    d.add_argument("--lr", type=float, default=6.0)
    d.add_argument("--seed", type=int, default=0)
    d.add_argument("--leak", type=float, default=1e-5)
    return p


def _load_batch(args, P):
    from .formats import read_array

    paths = args.logits.split(",")
    if len(paths) == 1:
        values = read_array(paths[0])
        if values.ndim != 3:
            raise UsageError(f"{paths[0]}: expected a (B, T, D) array, got {values.ndim} dimensions")
        B, T, _ = values.shape
        lengths = [T] * B
        if args.lengths:
            lengths = []
            for ln, line in enumerate(Path(args.lengths).read_text().splitlines(), 1):
                if line.strip():
                    try:
                        lengths.append(int(line.strip()))
                    except ValueError:
                        raise UsageError(f"{args.lengths}:{ln}: not an integer: {line.strip()!r}")
            if len(lengths) != B:
                raise UsageError(f"{args.lengths}: {len(lengths)} lengths for a batch of {B}")
            for b, n in enumerate(lengths):
                if not 1 <= n <= T:
                    raise UsageError(f"{args.lengths}: length {n} of item {b} not in [1, {T}]")
        return P.make_batch([values[b, :lengths[b]] for b in range(B)])
    if args.lengths:
        raise UsageError("--lengths is only valid with a single batched --logits file")
    seqs = []
    for path in paths:
        a = read_array(path)
        if a.ndim != 2:
            raise UsageError(f"{path}: expected a (T, D) array, got {a.ndim} dimensions")
        seqs.append(a)
    return P.make_batch(seqs)


def _load_graphs(args, batch, P):
    from .formats import parse_fst_text

    spec = Path(args.num_fsts)
    if spec.is_dir():
        files = sorted(spec.glob("*.fst"))
        if not files:
            raise UsageError(f"{spec}: no *.fst files found")
    else:
        files = [Path(s) for s in args.num_fsts.split(",")]
    if len(files) != batch.batch_size:
        raise UsageError(f"{len(files)} numerator graphs for a batch of {batch.batch_size}")
    D = batch.num_pdfs
    nums = [parse_fst_text(f.read_text(), D) for f in files]
    nums = [nums[i] for i in batch.order_map]
    den = parse_fst_text(Path(args.den_fst).read_text(), D)
    return P.ChainGraphBatch.from_graphs(nums), P.ChainGraphBatch.broadcast(den, batch.batch_size)


def _report(batch, res):
    inv = np.empty(batch.batch_size, dtype=np.int64)
    inv[batch.order_map] = np.arange(batch.batch_size)
    for i in range(batch.batch_size):
        n, d = res.per_utt[int(inv[i])]
        if math.isnan(n) or math.isnan(d):
            print(f"utt {i}: FAILED")
        else:
            print(f"utt {i}: num={n:.10f} den={d:.10f} F={n - d:.10f}")
    print(f"batch: F={res.objective:.10f} loss={res.loss:.10f} frames={batch.total_frames} "
          f"failed={res.num_failed}")


def _loss_or_grad(args) -> int:
    import paper_2005_09824_b200 as P

    batch = _load_batch(args, P)
    nums, den = _load_graphs(args, batch, P)
    try:
        res = P.chain_loss(batch, nums, den, P.FBOptions(leak_coefficient=args.leak),
                           normalize_by_frames=args.per_frame, precision=args.precision)
    except RuntimeError as exc:  # every utterance failed
        print(f"error: {exc}", file=sys.stderr)
        return 2
    _report(batch, res)
    if args.command == "grad":
        from .formats import write_array

        write_array(args.out, P.unsort(res.grad, batch.order_map))
        print(f"wrote {args.out}")
    return 2 if res.num_failed else 0


def _train_demo(args) -> int:
    from . import train

    r = train.train(num_phones=args.phones, num_utterances=args.utterances,
                    frames_per_phone=args.frames_per_phone, epochs=args.epochs,
                    learning_rate=args.lr, seed=args.seed, leak=args.leak)
    for e, loss in enumerate(r.losses):
        if e % max(1, len(r.losses) // 10) == 0 or e == len(r.losses) - 1:
            print(f"epoch {e}: loss={loss:.6f}")
    print(f"accuracy={r.accuracy:.4f} frames={r.total_frames} train_frames_per_s={r.frames_per_s:.0f}")
    return 0


def main(argv=None) -> int:
    try:
        args = _parser().parse_args(argv)
        if args.command == "train-demo":
            return _train_demo(args)
        return _loss_or_grad(args)
    except (UsageError, ValueError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
