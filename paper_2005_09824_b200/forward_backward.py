"""GPU forward-backward behind the reference's ``chainloss.forward_backward`` API.

Same public surface as /root/reference/pkg/src/chainloss/forward_backward.py:
``FBOptions``, ``ForwardResult``, ``FBResult``, ``forward``, ``backward``,
``occupation_posteriors``, ``forward_backward`` — same argument meaning,
same ``ValueError``s, per-item numerical failure reported as data.

Two device paths sit behind it:

* fused (``forward_backward(..., keep_trellis=False)``): one persistent-CTA
  launch per graph batch (``lfmmi_forward_backward``), fp32 by default;
* three-phase (``forward``/``backward``/``occupation_posteriors`` and
  ``keep_trellis=True``): the f64 parity kernels that mirror the numba seam
  (``lfmmi_{forward,backward,posterior}_kernel``) and materialise alpha/beta
  in the reference's (B, T+1, S_max) scaling convention.

There is no CPU fallback: without the extension or a GPU every call raises.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

from . import _backend
from .batching import LogLikBatch
from .graph import device_graphs

__all__ = [
    "FBOptions", "ForwardResult", "FBResult", "forward", "backward", "occupation_posteriors",
    "forward_backward", "set_precision", "get_precision", "forward_backward_device",
]

_PRECISION = os.environ.get("LFMMI_PRECISION", "fp32")


def set_precision(precision: str) -> None:
    """Default arithmetic of the fused path: ``"fp32"`` (production) or ``"fp64"``."""
    global _PRECISION
    if precision not in ("fp32", "fp64"):
        raise ValueError(f"precision must be 'fp32' or 'fp64', got {precision!r}")
    _PRECISION = precision


def get_precision() -> str:
    return _PRECISION


def _dtype(precision):
    import torch

    p = precision or _PRECISION
    if p not in ("fp32", "fp64"):
        raise ValueError(f"precision must be 'fp32' or 'fp64', got {p!r}")
    return torch.float32 if p == "fp32" else torch.float64


@dataclass(frozen=True)
class FBOptions:
    """Knobs of the recursion (forward_backward.py:40-60): leak coefficient,
    optional custom leak distribution (default uniform 1/S per graph), and the
    column-total floor below which an item is marked failed."""

    leak_coefficient: float = 1e-5
    leak_distribution: np.ndarray | None = None
    scale_floor: float = 1e-300

    def __post_init__(self) -> None:
        if not np.isfinite(self.leak_coefficient) or self.leak_coefficient < 0.0:
            raise ValueError(f"leak_coefficient must be >= 0, got {self.leak_coefficient}")
        if not np.isfinite(self.scale_floor) or self.scale_floor <= 0.0:
            raise ValueError(f"scale_floor must be positive, got {self.scale_floor}")


@dataclass
class ForwardResult:
    """Output of :func:`forward` (forward_backward.py:63-82)."""

    log_probs: np.ndarray
    alpha: np.ndarray
    scale_logs: np.ndarray
    failure_frames: np.ndarray
    emission_probs: np.ndarray
    frame_scales: np.ndarray


@dataclass
class FBResult:
    """Bundled forward-backward output (forward_backward.py:85-104)."""

    log_probs: np.ndarray
    posteriors: np.ndarray
    scale_logs: np.ndarray
    failure_frames: np.ndarray
    alpha: np.ndarray | None = None
    beta: np.ndarray | None = None

    @property
    def num_failed(self) -> int:
        return int(np.count_nonzero(self.failure_frames >= 0))


def _check_compatible(batch, graphs) -> None:
    """forward_backward.py:107-117."""
    if batch.batch_size != graphs.batch_size:
        raise ValueError(f"batch size mismatch: {batch.batch_size} sequences vs "
                         f"{graphs.batch_size} graphs")
    if batch.num_pdfs != graphs.num_pdfs:
        raise ValueError(f"pdf dimension mismatch: batch has {batch.num_pdfs}, "
                         f"graphs have {graphs.num_pdfs}")


def _leak_distribution(graphs, opts: FBOptions, explicit_uniform: bool = False):
    """forward_backward.py:133-166.  Returns None for the default uniform
    distribution (the kernels synthesise 1/S_g) unless ``explicit_uniform``."""
    custom = opts.leak_distribution
    if custom is None and not explicit_uniform:
        return None
    rows = graphs.final_probs.shape[0]
    s_max = graphs.max_states
    if custom is None:
        pi = np.zeros((rows, s_max), dtype=np.float64)
        for r in range(rows):
            n = graphs.item_num_states[0] if graphs.is_broadcast else graphs.item_num_states[r]
            pi[r, :n] = 1.0 / float(n)
        return pi
    arr = np.asarray(custom, dtype=np.float64)
    if arr.ndim == 1:
        arr = np.broadcast_to(arr, (graphs.batch_size, arr.shape[0]))
    if arr.shape != (graphs.batch_size, s_max):
        raise ValueError(f"leak_distribution must have shape ({graphs.batch_size}, {s_max}) "
                         f"or ({s_max},), got {np.asarray(custom).shape}")
    pi = np.zeros((rows, s_max), dtype=np.float64)
    for b in range(graphs.batch_size):
        n = int(graphs.item_num_states[b])
        row = arr[b]
        if np.any(row < 0.0) or np.any(row[n:] != 0.0):
            raise ValueError(f"leak_distribution item {b}: negative or padded-state mass")
        if abs(row[:n].sum() - 1.0) > 1e-12:
            raise ValueError(f"leak_distribution item {b}: must sum to 1")
        r = int(graphs.row_map[b])
        if np.any(pi[r] != 0.0) and not np.array_equal(pi[r], row):
            raise ValueError("broadcast graph batches require one shared leak_distribution")
        pi[r] = row
    return pi


# --------------------------------------------------------------- device core
_WORKSPACE: dict = {}


def _workspace(device, nbytes: int):
    """Scratch for one call, cached per (device, current stream): calls queued on
    one stream reuse it safely; calls on different streams never share it."""
    import torch

    key = (device.index, torch.cuda.current_stream(device).cuda_stream)
    buf = _WORKSPACE.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=device)
        _WORKSPACE[key] = buf
    return buf


def forward_backward_device(values, lengths, graphs, opts: FBOptions = FBOptions(), *,
                            posteriors=None, mode: int = 0, other_fail=None, total_frames=None,
                            want_scale_logs: bool = False):
    """Fused forward-backward on device tensors.

    ``values`` (B, T, D) CUDA float32/float64, ``lengths`` (B,) CUDA int32.
    Returns ``(posteriors, log_probs f64, fail_frames i32, scale_logs|None)``
    as CUDA tensors; no host synchronisation.
    """
    import torch

    ext = _backend.require_cuda()
    dev = values.device
    dg = device_graphs(graphs, dev)
    B, T, D = values.shape
    pi = _leak_distribution(graphs, opts)
    pi_t = None if pi is None else torch.as_tensor(pi, dtype=values.dtype, device=dev)
    if total_frames is None:
        total_frames = B * T  # upper bound; avoids a host sync on lengths
    prec = 1 if values.dtype == torch.float64 else 0
    ws = _workspace(dev, ext.workspace_size(dg.max_states, int(total_frames), prec))
    if posteriors is None:
        posteriors = torch.empty_like(values)
    logp = torch.empty(B, dtype=torch.float64, device=dev)
    fail = torch.empty(B, dtype=torch.int32, device=dev)
    sl = torch.empty((B, T), dtype=torch.float64, device=dev) if want_scale_logs else None
    ext.forward_backward(dg.handle, dg.row_map, values, lengths, float(opts.leak_coefficient),
                         float(opts.scale_floor), pi_t, int(total_frames), ws, posteriors,
                         int(mode), other_fail, logp, fail, sl)
    return posteriors, logp, fail, sl


_COPY_POOL = None


def _parallel_copy(dst: np.ndarray, src: np.ndarray) -> None:
    """dst[...] = src (with dtype conversion) in row chunks on a thread pool:
    numpy releases the GIL, so host memory bandwidth, not one core, bounds it."""
    global _COPY_POOL
    n = dst.shape[0]
    chunks = min(8, max(1, dst.nbytes >> 21), n)
    if chunks <= 1:
        np.copyto(dst, src, casting="unsafe")
        return
    if _COPY_POOL is None:
        from concurrent.futures import ThreadPoolExecutor

        _COPY_POOL = ThreadPoolExecutor(max_workers=8, thread_name_prefix="lfmmi-copy")
    cuts = np.linspace(0, n, chunks + 1).astype(np.int64)
    futs = [_COPY_POOL.submit(np.copyto, dst[a:b], src[a:b], casting="unsafe")
            for a, b in zip(cuts[:-1], cuts[1:]) if b > a]
    for f in futs:
        f.result()


def _to_device(batch, dtype):
    """Host batch -> device (values in ``dtype``, lengths int32).

    The numpy values are staged into pinned host memory already converted to
    ``dtype`` (parallel chunked copy), then copied asynchronously: for fp32
    half the PCIe bytes of the f64 array and no pageable bounce buffer.
    """
    import torch

    dev = torch.device("cuda", torch.cuda.current_device())
    src = np.asarray(batch.values)
    host = torch.empty(src.shape, dtype=dtype, pin_memory=True)
    _parallel_copy(host.numpy().reshape(src.shape[0], -1), src.reshape(src.shape[0], -1))
    values = host.to(dev, non_blocking=True)
    lens = torch.from_numpy(np.asarray(batch.lengths, dtype=np.int32)).pin_memory()
    lengths = lens.to(dev, non_blocking=True)
    return dev, values, lengths


def _to_host_f64(t):
    """Device tensor -> float64 numpy array through pinned memory (one async
    D2H, returned as a view of the pinned buffer: no second host copy)."""
    import torch

    out = torch.empty(t.shape, dtype=torch.float64, pin_memory=True)
    out.copy_(t.to(torch.float64), non_blocking=True)
    return out


# ------------------------------------------------------ three-phase (parity)
def _emissions_device(values, lengths_np):
    """forward_backward.py:120-130 on device: per-frame max shift + exp, padding zero."""
    import torch

    B, T, _ = values.shape
    valid = torch.arange(T, device=values.device)[None, :] < torch.as_tensor(
        lengths_np, device=values.device)[:, None]
    m = values.max(dim=2).values
    m = torch.where(valid, m, torch.zeros_like(m))
    expl = torch.exp(values - m[:, :, None]) * valid[:, :, None]
    return expl.contiguous(), m


def forward(batch: LogLikBatch, graphs, opts: FBOptions = FBOptions()) -> ForwardResult:
    """Forward recursion (forward_backward.py:169-221) via the f64 parity kernel."""
    import torch

    _check_compatible(batch, graphs)
    ext = _backend.require_cuda()
    dev, values, lengths = _to_device(batch, torch.float64)
    dg = device_graphs(graphs, dev)
    expl, shifts = _emissions_device(values, batch.lengths)
    pi = torch.as_tensor(_leak_distribution(graphs, opts, explicit_uniform=True), device=dev)
    B, T, _ = values.shape
    S = int(graphs.max_states)
    alpha = torch.zeros((B, T + 1, S), dtype=torch.float64, device=dev)
    scales = torch.ones((B, T), dtype=torch.float64, device=dev)
    fail = torch.full((B,), -1, dtype=torch.int64, device=dev)
    ext.forward_kernel(dg.handle, dg.row_map, expl, lengths, float(opts.leak_coefficient), pi,
                       float(opts.scale_floor), alpha, scales, fail)
    scale_logs = (torch.log(scales) + shifts).cpu().numpy()
    fail_np = fail.cpu().numpy()
    log_probs = np.empty(B, dtype=np.float64)
    for b in range(B):
        log_probs[b] = np.nan if fail_np[b] >= 0 else scale_logs[b, : batch.lengths[b]].sum()
    return ForwardResult(log_probs=log_probs, alpha=alpha.cpu().numpy(), scale_logs=scale_logs,
                         failure_frames=fail_np, emission_probs=expl.cpu().numpy(),
                         frame_scales=scales.cpu().numpy())


def backward(batch: LogLikBatch, graphs, opts: FBOptions, fwd: ForwardResult) -> np.ndarray:
    """Backward recursion (forward_backward.py:224-256) via the f64 parity kernel."""
    import torch

    _check_compatible(batch, graphs)
    ext = _backend.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    dg = device_graphs(graphs, dev)
    pi = torch.as_tensor(_leak_distribution(graphs, opts, explicit_uniform=True), device=dev)
    as_dev = lambda a, dt=torch.float64: torch.as_tensor(np.ascontiguousarray(a), device=dev).to(dt)  # noqa: E731
    beta = torch.zeros(np.shape(fwd.alpha), dtype=torch.float64, device=dev)
    ext.backward_kernel(dg.handle, dg.row_map, as_dev(fwd.emission_probs),
                        as_dev(batch.lengths, torch.int32), as_dev(fwd.frame_scales),
                        float(opts.leak_coefficient), pi,
                        as_dev(fwd.failure_frames, torch.int64), beta)
    return beta.cpu().numpy()


def occupation_posteriors(batch: LogLikBatch, graphs, fwd: ForwardResult,
                          beta: np.ndarray) -> np.ndarray:
    """Occupation posteriors (forward_backward.py:259-287) via the f64 parity kernel."""
    import torch

    _check_compatible(batch, graphs)
    ext = _backend.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    dg = device_graphs(graphs, dev)
    as_dev = lambda a, dt=torch.float64: torch.as_tensor(np.ascontiguousarray(a), device=dev).to(dt)  # noqa: E731
    gamma = torch.zeros(np.shape(batch.values), dtype=torch.float64, device=dev)
    ext.posterior_kernel(dg.handle, dg.row_map, as_dev(fwd.emission_probs),
                         as_dev(batch.lengths, torch.int32), as_dev(fwd.alpha), as_dev(beta),
                         as_dev(fwd.failure_frames, torch.int64), gamma)
    return gamma.cpu().numpy()


def forward_backward(batch: LogLikBatch, graphs, opts: FBOptions = FBOptions(),
                     keep_trellis: bool = False, precision: str | None = None) -> FBResult:
    """Forward pass, backward pass and posteriors (forward_backward.py:290-307).

    ``keep_trellis=True`` runs the three f64 parity kernels and returns alpha
    and beta; otherwise one fused launch at ``precision`` (default
    :func:`get_precision`).
    """
    if keep_trellis:
        fwd = forward(batch, graphs, opts)
        beta = backward(batch, graphs, opts, fwd)
        gamma = occupation_posteriors(batch, graphs, fwd, beta)
        return FBResult(fwd.log_probs, gamma, fwd.scale_logs, fwd.failure_frames, fwd.alpha, beta)
    _check_compatible(batch, graphs)
    _backend.require_cuda()
    dev, values, lengths = _to_device(batch, _dtype(precision))
    post, logp, fail, sl = forward_backward_device(values, lengths, graphs, opts,
                                                   total_frames=batch.total_frames,
                                                   want_scale_logs=True)
    post_h = _to_host_f64(post)
    import torch

    torch.cuda.current_stream(dev).synchronize()
    return FBResult(log_probs=logp.cpu().numpy(), posteriors=post_h.numpy(),
                    scale_logs=sl.cpu().numpy(),
                    failure_frames=fail.cpu().numpy().astype(np.int64))
