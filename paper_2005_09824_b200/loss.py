"""LF-MMI objective: drop-in ``chain_loss`` plus the paper's torch API.

* :func:`chain_loss` — same signature, result type and failure semantics as
  /root/reference/pkg/src/chainloss/loss.py:42-84 (numpy in, numpy out,
  sorted batch order, ``RuntimeError`` when every utterance fails).  One C-ABI
  call (``lfmmi_chain_loss``): the numerator pass (warp per utterance) runs on
  an auxiliary stream concurrently with the denominator pass (CTA per
  utterance, writes -gamma_den into the gradient); a combine step adds
  gamma_num and a tiny reduction produces {objective, frames, failed}.
* :func:`chain_loss_device` — the same on CUDA tensors, no host sync.
* :class:`ChainFunction` / :class:`ChainLoss` — the paper's
  ``autograd.Function`` / ``nn.Module``.  With a process group
  the three scalar totals are all-reduced (NCCL over NVLink) so the
  normalised loss equals the single-GPU one; gradients are never exchanged.
"""

from __future__ import annotations

import collections
from dataclasses import dataclass

import numpy as np

from . import _backend
from .forward_backward import (FBOptions, _check_compatible, _dtype, _leak_distribution,
                               _to_device, _to_host_f64, _workspace)
from .graph import ChainGraphBatch, device_graphs

__all__ = ["ChainLossResult", "chain_loss", "chain_loss_device", "chain_loss_packed",
           "ChainFunction", "ChainLoss"]


@dataclass
class ChainLossResult:
    """Objective, loss and gradient of one batch, in sorted batch order (loss.py:22-39)."""

    objective: float
    loss: float
    grad: np.ndarray
    per_utt: list
    num_failed: int


def chain_loss_device(values, lengths, numerators, denominator, opts: FBOptions = FBOptions(), *,
                      total_frames=None, grad=None):
    """LF-MMI on device tensors.

    ``values`` (B, T, D) CUDA float32/float64; ``lengths`` (B,) CUDA int32.
    Returns ``(grad, num_logp, den_logp, num_fail, den_fail, totals)`` where
    ``grad = gamma_num - gamma_den`` (zero rows for failed / padded frames)
    and ``totals = [sum_ok(num - den), sum_ok T_b, #failed]`` (f64).
    """
    import torch

    ext = _backend.require_cuda()
    dev = values.device
    B, T, D = values.shape
    _check_batch(numerators, B, "numerators")
    _check_batch(denominator, B, "denominator")
    pn = _leak_distribution(numerators, opts)
    pd = _leak_distribution(denominator, opts)
    ng = device_graphs(numerators, dev, linear_ok=values.dtype == torch.float32 and pn is None)
    dgr = device_graphs(denominator, dev)
    pn = None if pn is None else torch.as_tensor(pn, dtype=values.dtype, device=dev)
    pd = None if pd is None else torch.as_tensor(pd, dtype=values.dtype, device=dev)
    if total_frames is None:
        total_frames = B * T
    prec = 1 if values.dtype == torch.float64 else 0
    ws = _workspace(dev, ext.chain_loss_workspace_size(ng.handle, dgr.handle, B, T, D,
                                                       int(total_frames), prec))
    if grad is None:
        grad = torch.empty_like(values)
    f64 = dict(dtype=torch.float64, device=dev)
    i32 = dict(dtype=torch.int32, device=dev)
    num_lp, den_lp = torch.empty(B, **f64), torch.empty(B, **f64)
    num_fail, den_fail = torch.empty(B, **i32), torch.empty(B, **i32)
    totals = torch.empty(3, **f64)
    ext.chain_loss(ng.handle, ng.row_map, dgr.handle, dgr.row_map, values, lengths,
                   float(opts.leak_coefficient), float(opts.scale_floor), pn, pd,
                   int(total_frames), ws, grad,
                   num_lp, den_lp, num_fail, den_fail, totals)
    return grad, num_lp, den_lp, num_fail, den_fail, totals


def chain_loss_packed(values, lengths, numerators, denominator, opts: FBOptions = FBOptions(), *,
                      max_frames: int | None = None, total_frames: int | None = None, grad=None):
    """LF-MMI on a ragged (packed) batch — device-side batching.

    ``values`` (sum_b T_b, D) CUDA float32/float64 with utterance b's frames at
    rows ``[sum_{j<b} T_j, sum_{j<=b} T_j)``; ``lengths`` (B,) CUDA int32, any
    order (no host sort, no padding: replaces make_batch, batching.py:52-97);
    ``numerators`` aligned with ``lengths``.  Returns the same tuple as
    :func:`chain_loss_device` with ``grad`` in the packed layout (caller order).
    Uniform leak distribution.  ``max_frames`` / ``total_frames`` default to a
    host read of ``lengths``.
    """
    import torch

    ext = _backend.require_cuda()
    dev = values.device
    if values.dim() != 2:
        raise ValueError(f"packed values must be (sum T, D), got {tuple(values.shape)}")
    if opts.leak_distribution is not None:
        raise ValueError("chain_loss_packed supports the uniform leak distribution only")
    B = int(lengths.shape[0])
    N, D = values.shape
    if max_frames is None or total_frames is None:
        lens = lengths.cpu()
        max_frames = int(lens.max()) if max_frames is None else max_frames
        total_frames = int(lens.sum()) if total_frames is None else total_frames
    if total_frames != N:
        raise ValueError(f"sum of lengths {total_frames} != packed rows {N}")
    denominator = _as_graph_batch(denominator, B)
    _check_batch(numerators, B, "numerators")
    _check_batch(denominator, B, "denominator")
    # a list of numerator graphs goes straight to the per-utterance linear
    # records (no padded ChainGraphBatch build)
    ng = device_graphs(numerators, dev, linear_ok=values.dtype == torch.float32)
    dgr = device_graphs(denominator, dev)
    if ng.num_pdfs != D or dgr.num_pdfs != D:
        raise ValueError(f"pdf dimension mismatch: values have {D}, graphs have "
                         f"{ng.num_pdfs}/{dgr.num_pdfs}")
    prec = 1 if values.dtype == torch.float64 else 0
    ws = _workspace(dev, ext.chain_loss_workspace_size(ng.handle, dgr.handle, B, int(max_frames),
                                                       int(D), int(total_frames), prec))
    if grad is None:
        grad = torch.empty_like(values)
    f64 = dict(dtype=torch.float64, device=dev)
    i32 = dict(dtype=torch.int32, device=dev)
    num_lp, den_lp = torch.empty(B, **f64), torch.empty(B, **f64)
    num_fail, den_fail = torch.empty(B, **i32), torch.empty(B, **i32)
    totals = torch.empty(3, **f64)
    ext.chain_loss_packed(ng.handle, ng.row_map, dgr.handle, dgr.row_map, values, lengths,
                          int(max_frames), float(opts.leak_coefficient), float(opts.scale_floor),
                          int(total_frames), ws, grad, num_lp, den_lp, num_fail, den_fail, totals)
    return grad, num_lp, den_lp, num_fail, den_fail, totals


def chain_loss(batch, numerators, denominator, opts: FBOptions = FBOptions(),
               normalize_by_frames: bool = True, precision: str | None = None) -> ChainLossResult:
    """MMI objective and gradient for one batch (loss.py:42-84), computed on the GPU."""
    _check_compatible(batch, numerators)
    _check_compatible(batch, denominator)
    _backend.require_cuda()
    dev, values, lengths = _to_device(batch, _dtype(precision))
    import torch

    grad, num_lp, den_lp, num_fail, den_fail, totals = chain_loss_device(
        values, lengths, numerators, denominator, opts, total_frames=batch.total_frames)
    # one read-back: totals + per-utterance log-probs, then the gradient (f64,
    # the reference's dtype) into pinned memory; a single synchronisation
    small = torch.cat([totals, num_lp, den_lp]).to("cpu", non_blocking=True)
    grad_h = _to_host_f64(grad)
    torch.cuda.current_stream(dev).synchronize()
    small = small.numpy()
    tot, nl, dl = small[:3], small[3:3 + batch.batch_size], small[3 + batch.batch_size:]
    num_failed = int(round(tot[2]))
    if num_failed == batch.batch_size:
        raise RuntimeError(f"all {batch.batch_size} utterances failed numerically")
    objective = float(tot[0])
    frames = int(round(tot[1]))
    loss = -objective / frames if normalize_by_frames else -objective
    per_utt = [(float(nl[b]), float(dl[b])) for b in range(batch.batch_size)]
    return ChainLossResult(objective=objective, loss=loss, grad=grad_h.numpy(), per_utt=per_utt,
                           num_failed=num_failed)


def _check_batch(graphs, batch_size, what):
    """The device code indexes ``row_map[b]`` for every item: sizes must agree."""
    n = len(graphs) if isinstance(graphs, (list, tuple)) else getattr(graphs, "batch_size", None)
    if n is not None and int(n) != int(batch_size):
        raise ValueError(f"{what} batch has {n} items, input has {batch_size}")


# ------------------------------------------------------------------- torch API
def _as_graph_batch(graphs, batch_size):
    if isinstance(graphs, (list, tuple)):
        return ChainGraphBatch.from_graphs(graphs)
    if hasattr(graphs, "forward_from") and not hasattr(graphs, "row_map"):  # a single ChainGraph
        return ChainGraphBatch.broadcast(graphs, batch_size)
    return graphs


def _autograd_function():
    import torch

    class _ChainFunction(torch.autograd.Function):
        """LF-MMI loss as an autograd function (paper's ``ChainFunction``).

        ``apply(input, input_lengths, numerators, denominator, opts,
        normalize_by_frames, process_group)`` -> scalar loss
        ``-sum_ok(logP_num - logP_den) / frames`` (or un-normalised).
        ``input`` is (B, T, D) on CUDA in any length order — or ragged
        (sum_b T_b, D) with ``input_lengths`` giving the split; ``numerators``
        is aligned with it.  Backward returns ``-(gamma_num - gamma_den) / frames``
        scaled by the incoming gradient.
        """

        @staticmethod
        def forward(ctx, input, input_lengths, numerators, denominator, opts=FBOptions(),
                    normalize_by_frames=True, process_group=None):
            if not input.is_cuda:
                raise _backend.BackendUnavailable("ChainFunction needs a CUDA input tensor")
            x = input.detach().contiguous()
            if x.dtype not in (torch.float32, torch.float64):
                x = x.float()
            lengths = input_lengths.to(device=x.device, dtype=torch.int32).contiguous()
            B = lengths.shape[0]
            # numerator lists stay lists (per-utterance linear records) unless a
            # custom leak distribution needs the padded batch view
            nums = (numerators if opts.leak_distribution is None and isinstance(numerators, (list, tuple))
                    else _as_graph_batch(numerators, B))
            den = _as_graph_batch(denominator, B)
            if x.dim() == 2:  # ragged (sum T, D) input: device-side batching
                grad, _, _, _, _, totals = chain_loss_packed(x, lengths, nums, den, opts)
            else:
                grad, _, _, _, _, totals = chain_loss_device(x, lengths, nums, den, opts)
            if process_group is not None:
                import torch.distributed as dist

                dist.all_reduce(totals, op=dist.ReduceOp.SUM, group=process_group)
            if normalize_by_frames:
                # every utterance failed => no frames: zero loss and gradient
                # (not 0 * inf = NaN into the model), no host sync
                frames = totals[1]
                scale = torch.where(frames > 0, 1.0 / frames.clamp_min(1.0), frames.new_zeros(()))
            else:
                scale = totals.new_ones(())
            loss = -totals[0] * scale
            ctx.save_for_backward(grad, scale)
            ctx.in_dtype = input.dtype
            return loss.to(input.dtype)

        @staticmethod
        def backward(ctx, grad_output):
            grad, scale = ctx.saved_tensors
            g = grad * (-(grad_output.to(torch.float64) * scale)).to(grad.dtype)
            return g.to(ctx.in_dtype), None, None, None, None, None, None

    return _ChainFunction


class _LazyFunction:
    _fn = None

    def __getattr__(self, name):
        if _LazyFunction._fn is None:
            _LazyFunction._fn = _autograd_function()
        return getattr(_LazyFunction._fn, name)


ChainFunction = _LazyFunction()


def _module_base():
    import torch

    return torch.nn.Module


class ChainLoss(_module_base()):
    """``nn.Module`` wrapper (paper's ``ChainLoss``): holds the denominator graph.

    ``ChainLoss(den_graph, opts=FBOptions(), normalize_by_frames=True,
    process_group=None)(input, input_lengths, num_graphs)`` -> scalar loss.
    """

    def __init__(self, den_graph, opts: FBOptions = FBOptions(), normalize_by_frames: bool = True,
                 process_group=None):
        super().__init__()
        self.den_graph = den_graph
        self.opts = opts
        self.normalize_by_frames = normalize_by_frames
        self.process_group = process_group
        self._den_cache = collections.OrderedDict()

    def _den_batch(self, batch_size):
        if hasattr(self.den_graph, "row_map"):
            return self.den_graph
        den = self._den_cache.pop(batch_size, None)
        if den is None:
            den = ChainGraphBatch.broadcast(self.den_graph, batch_size)
        self._den_cache[batch_size] = den  # most recent last; a few batch sizes at most
        while len(self._den_cache) > 4:
            self._den_cache.popitem(last=False)
        return den

    def forward(self, input, input_lengths, num_graphs):
        # B = number of utterances (input may be ragged (sum T, D))
        den = self._den_batch(int(input_lengths.shape[0]))
        return ChainFunction.apply(input, input_lengths, num_graphs, den, self.opts,
                                   self.normalize_by_frames, self.process_group)
