"""TEST INFRASTRUCTURE ONLY — CPU oracle for the LF-MMI hot path.

This module is the parity checker.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference`` fallback)
may import it; the product package never does, and fails loudly when its CUDA
extension is missing instead of falling back here.

It restates the reference algorithm (chainloss 0.1.0,
``/root/reference/pkg/src/chainloss``) on the CPU:

* the three recursions are compiled C (``oracle/lfmmi_oracle.c``), a sequential
  fp64 transliteration of the numba kernels in ``_kernels.py:54-224``;
* the host orchestration below mirrors ``forward_backward.py:120-307`` and
  ``loss.py:42-84`` line for line (numpy emissions, uniform/custom leak
  distribution, log-probability assembly, num-minus-den combination).

Parity status: **pinned** — ``tests/test_oracle_golden.py`` checks this module
bit-for-bit against golden vectors recorded from the reference itself
(``tests/golden/make_golden.py``).

Graph and batch arguments are duck-typed: anything exposing the reference's
``ChainGraphBatch`` / ``LogLikBatch`` attribute names works, i.e. both the
reference objects and ``paper_2005_09824_b200``'s drop-in classes.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liblfmmi_oracle.so")
_lib = None


def build() -> str:
    """Compile the C restatement (``oracle/Makefile``) if needed."""
    src = os.path.join(_HERE, "lfmmi_oracle.c")
    if (not os.path.exists(_LIB_PATH)) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        I = ctypes.c_int64
        D = ctypes.c_double
        lib.oracle_forward.argtypes = [P] * 10 + [D, P, D] + [I] * 6 + [P, P, P]
        lib.oracle_backward.argtypes = [P] * 10 + [D, P, P] + [I] * 6 + [P]
        lib.oracle_posterior.argtypes = [P] * 11 + [I] * 5 + [P]
        for fn in (lib.oracle_forward, lib.oracle_backward, lib.oracle_posterior):
            fn.restype = None
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous"
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# ---------------------------------------------------------------- kernels
def forward_kernel(expl, lengths, bvalid, row_map, bw_from, bw_pdf, bw_prob, bw_index,
                   final_probs, init_states, leak, leak_pi, scale_floor, alpha, scales,
                   fail_frames):
    """Same signature and in-place contract as ``_kernels.py:54`` forward_kernel."""
    lib = _load()
    expl = _c(expl, np.float64)
    B, T, D = expl.shape
    G, I = bw_from.shape
    S = alpha.shape[2]
    args = [_c(lengths, np.int64), _c(bvalid, np.int64), _c(row_map, np.int64),
            _c(bw_from, np.uint32), _c(bw_pdf, np.uint32), _c(bw_prob, np.float64),
            _c(bw_index, np.uint32), _c(final_probs, np.float64), _c(init_states, np.uint32)]
    pi = _c(leak_pi, np.float64)
    lib.oracle_forward(_p(expl), *[_p(a) for a in args], float(leak), _p(pi),
                       float(scale_floor), B, T, D, G, I, S, _p(alpha), _p(scales),
                       _p(fail_frames))


def backward_kernel(expl, lengths, bvalid, row_map, fw_to, fw_pdf, fw_prob, fw_index,
                    final_probs, scales, leak, leak_pi, fail_frames, beta):
    """Same signature and in-place contract as ``_kernels.py:125`` backward_kernel."""
    lib = _load()
    expl = _c(expl, np.float64)
    B, T, D = expl.shape
    G, I = fw_to.shape
    S = beta.shape[2]
    args = [_c(lengths, np.int64), _c(bvalid, np.int64), _c(row_map, np.int64),
            _c(fw_to, np.uint32), _c(fw_pdf, np.uint32), _c(fw_prob, np.float64),
            _c(fw_index, np.uint32), _c(final_probs, np.float64), _c(scales, np.float64)]
    pi = _c(leak_pi, np.float64)
    fail = _c(fail_frames, np.int64)
    lib.oracle_backward(_p(expl), *[_p(a) for a in args], float(leak), _p(pi), _p(fail),
                        B, T, D, G, I, S, _p(beta))


def posterior_kernel(expl, lengths, row_map, item_ntrans, fw_from, fw_to, fw_pdf, fw_prob,
                     alpha, beta, fail_frames, gamma):
    """Same signature and in-place contract as ``_kernels.py:194`` posterior_kernel."""
    lib = _load()
    expl = _c(expl, np.float64)
    B, T, D = expl.shape
    G, I = fw_from.shape
    S = alpha.shape[2]
    args = [_c(lengths, np.int64), _c(row_map, np.int64), _c(item_ntrans, np.int64),
            _c(fw_from, np.uint32), _c(fw_to, np.uint32), _c(fw_pdf, np.uint32),
            _c(fw_prob, np.float64), _c(alpha, np.float64), _c(beta, np.float64),
            _c(fail_frames, np.int64)]
    lib.oracle_posterior(_p(expl), *[_p(a) for a in args], B, T, D, I, S, _p(gamma))


# ---------------------------------------------------------- orchestration
@dataclass
class OracleForward:
    log_probs: np.ndarray
    alpha: np.ndarray
    scale_logs: np.ndarray
    failure_frames: np.ndarray
    emission_probs: np.ndarray
    frame_scales: np.ndarray


@dataclass
class OracleFB:
    log_probs: np.ndarray
    posteriors: np.ndarray
    scale_logs: np.ndarray
    failure_frames: np.ndarray
    alpha: np.ndarray | None = None
    beta: np.ndarray | None = None


@dataclass
class OracleLoss:
    objective: float
    loss: float
    grad: np.ndarray
    per_utt: list
    num_failed: int


def emissions(values, lengths):
    """``forward_backward.py:120-130`` _emissions."""
    values = np.asarray(values, dtype=np.float64)
    expl = np.zeros_like(values)
    shifts = np.zeros(values.shape[:2], dtype=np.float64)
    for b in range(values.shape[0]):
        n = int(lengths[b])
        valid = values[b, :n]
        m = valid.max(axis=1)
        shifts[b, :n] = m
        np.exp(valid - m[:, None], out=expl[b, :n])
    return expl, shifts


def leak_distribution(graphs, leak_distribution=None):
    """``forward_backward.py:133-166`` _leak_distribution (uniform or custom)."""
    rows = graphs.final_probs.shape[0]
    s_max = graphs.max_states
    if leak_distribution is None:
        pi = np.zeros((rows, s_max), dtype=np.float64)
        for r in range(rows):
            n = graphs.item_num_states[0] if graphs.is_broadcast else graphs.item_num_states[r]
            pi[r, :n] = 1.0 / float(n)
        return pi
    arr = np.asarray(leak_distribution, dtype=np.float64)
    if arr.ndim == 1:
        arr = np.broadcast_to(arr, (graphs.batch_size, arr.shape[0]))
    pi = np.zeros((rows, s_max), dtype=np.float64)
    for b in range(graphs.batch_size):
        pi[int(graphs.row_map[b])] = arr[b]
    return pi


def forward(batch, graphs, leak=1e-5, leak_dist=None, scale_floor=1e-300) -> OracleForward:
    """``forward_backward.py:169-221`` forward."""
    expl, shifts = emissions(batch.values, batch.lengths)
    pi = leak_distribution(graphs, leak_dist)
    B, T = expl.shape[:2]
    S = graphs.max_states
    alpha = np.zeros((B, T + 1, S))
    scales = np.ones((B, T))
    fail = np.full(B, -1, dtype=np.int64)
    forward_kernel(expl, batch.lengths, batch.valid_batch_sizes, graphs.row_map,
                   graphs.backward_from, graphs.backward_pdf, graphs.backward_probs,
                   graphs.backward_index, graphs.final_probs, graphs.initial_states,
                   leak, pi, scale_floor, alpha, scales, fail)
    scale_logs = np.log(scales) + shifts
    log_probs = np.empty(B)
    for b in range(B):
        log_probs[b] = np.nan if fail[b] >= 0 else scale_logs[b, : batch.lengths[b]].sum()
    return OracleForward(log_probs, alpha, scale_logs, fail, expl, scales)


def backward(batch, graphs, fwd: OracleForward, leak=1e-5, leak_dist=None) -> np.ndarray:
    """``forward_backward.py:224-256`` backward."""
    pi = leak_distribution(graphs, leak_dist)
    beta = np.zeros_like(fwd.alpha)
    backward_kernel(fwd.emission_probs, batch.lengths, batch.valid_batch_sizes,
                    graphs.row_map, graphs.forward_to, graphs.forward_pdf,
                    graphs.forward_probs, graphs.forward_index, graphs.final_probs,
                    fwd.frame_scales, leak, pi, fwd.failure_frames, beta)
    return beta


def occupation_posteriors(batch, graphs, fwd: OracleForward, beta) -> np.ndarray:
    """``forward_backward.py:259-287`` occupation_posteriors."""
    gamma = np.zeros(np.shape(batch.values))
    posterior_kernel(fwd.emission_probs, batch.lengths, graphs.row_map,
                     graphs.item_num_transitions, graphs.forward_from, graphs.forward_to,
                     graphs.forward_pdf, graphs.forward_probs, fwd.alpha, beta,
                     fwd.failure_frames, gamma)
    return gamma


def forward_backward(batch, graphs, leak=1e-5, leak_dist=None, scale_floor=1e-300,
                     keep_trellis=False) -> OracleFB:
    """``forward_backward.py:290-307`` forward_backward."""
    fwd = forward(batch, graphs, leak, leak_dist, scale_floor)
    beta = backward(batch, graphs, fwd, leak, leak_dist)
    gamma = occupation_posteriors(batch, graphs, fwd, beta)
    return OracleFB(fwd.log_probs, gamma, fwd.scale_logs, fwd.failure_frames,
                    fwd.alpha if keep_trellis else None, beta if keep_trellis else None)


def chain_loss(batch, numerators, denominator, leak=1e-5, leak_dist=None,
               scale_floor=1e-300, normalize_by_frames=True) -> OracleLoss:
    """``loss.py:42-84`` chain_loss."""
    num = forward_backward(batch, numerators, leak, leak_dist, scale_floor)
    den = forward_backward(batch, denominator, leak, leak_dist, scale_floor)
    failed = (num.failure_frames >= 0) | (den.failure_frames >= 0)
    ok = ~failed
    if not ok.any():
        raise RuntimeError(f"all {len(failed)} utterances failed numerically")
    objective = float((num.log_probs[ok] - den.log_probs[ok]).sum())
    grad = num.posteriors - den.posteriors
    if failed.any():
        grad[failed] = 0.0
    frames = int(np.asarray(batch.lengths)[ok].sum())
    loss = -objective / frames if normalize_by_frames else -objective
    per_utt = [(float(num.log_probs[b]), float(den.log_probs[b])) for b in range(len(failed))]
    return OracleLoss(objective, loss, grad, per_utt, int(np.count_nonzero(failed)))
