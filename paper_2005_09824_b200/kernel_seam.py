"""The reference's kernel seam, bound to the C-ABI through ctypes.

``chainloss.forward_backward`` resolves ``_kernels.forward_kernel``,
``_kernels.backward_kernel`` and ``_kernels.posterior_kernel`` at call time
(/root/reference/pkg/src/chainloss/forward_backward.py:25,187,240,273), so
rebinding those three module attributes moves the reference's own
orchestration onto the GPU without touching any other line of it.  This
module provides drop-in replacements with the numba signatures
(``_kernels.py:54-72,125-141,194-208``) and in-place output contract: the
caller's numpy arrays are uploaded, ``lfmmi_{forward,backward,posterior}_kernel``
(include/lfmmi.h; the exact-order f64 parity kernels) run on the current CUDA
device, and the results are copied back into the caller's arrays.

It is exactly the binding INTEGRATION.md shows a reference maintainer adding
(``ctypes`` on ``libpaper_lfmmi.so``; device memory from torch, which is
plumbing here).  :func:`install` / :func:`uninstall` do the rebinding.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _backend

__all__ = ["forward_kernel", "backward_kernel", "posterior_kernel", "install", "uninstall",
           "library"]

_LIB = None
_HANDLES: dict = {}
_SAVED: dict = {}
CALLS = {"forward_kernel": 0, "backward_kernel": 0, "posterior_kernel": 0}  # seam traffic


def library() -> ctypes.CDLL:
    """ctypes view of ``libpaper_lfmmi.so`` with the include/lfmmi.h prototypes."""
    global _LIB
    if _LIB is None:
        _backend.require_cuda()
        lib = ctypes.CDLL(_backend.core_library_path())
        P, I32, I64, D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        lib.lfmmi_last_error.restype = ctypes.c_char_p
        lib.lfmmi_graphs_create.argtypes = [I32, I32, I32, I32] + [P] * 12 + [ctypes.POINTER(P)]
        lib.lfmmi_graphs_destroy.argtypes = [P]
        lib.lfmmi_forward_kernel.argtypes = [P, P, I32, I32, I32, P, P, D, P, D, P, P, P, P]
        lib.lfmmi_backward_kernel.argtypes = [P, P, I32, I32, I32, P, P, P, D, P, P, P, P]
        lib.lfmmi_posterior_kernel.argtypes = [P, P, I32, I32, I32, P, P, P, P, P, P, P]
        for f in (lib.lfmmi_graphs_create, lib.lfmmi_graphs_destroy, lib.lfmmi_forward_kernel,
                  lib.lfmmi_backward_kernel, lib.lfmmi_posterior_kernel):
            f.restype = ctypes.c_int
        _LIB = lib
    return _LIB


def _check(rc: int) -> None:
    if rc != 0:
        msg = library().lfmmi_last_error().decode()
        raise (ValueError if rc == 1 else RuntimeError)(f"lfmmi status {rc}: {msg}")


def _hp(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


def _from_ranges(index: np.ndarray, num_arcs: np.ndarray, i_max: int) -> np.ndarray:
    """Per-arc owning state of a (G, S, 2) range table (the implicit column)."""
    G, S, _ = index.shape
    out = np.zeros((G, i_max), dtype=np.uint32)
    for g in range(G):
        for s in range(S):
            lo, hi = int(index[g, s, 0]), int(index[g, s, 1])
            out[g, lo:hi] = s
    return out


def _graph_handle(kind: str, key_arrays: tuple, build):
    """Create (once) the device graph pack behind a set of immutable reference arrays."""
    key = (kind,) + tuple((id(a), a.ctypes.data, a.shape) for a in key_arrays)
    hit = _HANDLES.get(key)
    if hit is None:
        if len(_HANDLES) >= 32:  # bounded cache
            old_key = next(iter(_HANDLES))
            library().lfmmi_graphs_destroy(_HANDLES.pop(old_key)[0])
        hit = (build(), key_arrays)  # keep the arrays alive so ids stay unique
        _HANDLES[key] = hit
    return hit[0]


def _create(G, S, I, D, num_arcs, fw, bw, finals, inits):
    lib = library()
    row_s = np.full(G, S, dtype=np.int64)  # padded states carry no arcs, pi = 0, final = 0
    row_i = np.ascontiguousarray(num_arcs, dtype=np.int64)
    u32 = lambda a: None if a is None else np.ascontiguousarray(a, dtype=np.uint32)  # noqa: E731
    f64 = lambda a: None if a is None else np.ascontiguousarray(a, dtype=np.float64)  # noqa: E731
    arrs = [u32(fw[0]), u32(fw[1]), u32(fw[2]), f64(fw[3])]
    arrs += [u32(bw[0]), u32(bw[1]), u32(bw[2]), f64(bw[3])] if bw else [None] * 4
    fin = f64(finals)
    ini = u32(inits)
    out = ctypes.c_void_p()
    _check(lib.lfmmi_graphs_create(G, S, max(I, 1), D, _hp(row_s), _hp(row_i),
                                   *[_hp(a) for a in arrs], _hp(fin), _hp(ini),
                                   ctypes.byref(out)))
    return out.value


def _dev(a, dtype):
    import torch

    return torch.as_tensor(np.ascontiguousarray(a), device="cuda").to(dtype)


def _stream():
    import torch

    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _copy_back(dst: np.ndarray, t) -> None:
    import torch

    torch.cuda.synchronize()
    np.copyto(dst, t.cpu().numpy().astype(dst.dtype, copy=False))


def forward_kernel(expl, lengths, bvalid, row_map, bw_from, bw_pdf, bw_prob, bw_index,
                   final_probs, init_states, leak, leak_pi, scale_floor, alpha, scales,
                   fail_frames):
    """``_kernels.forward_kernel`` (_kernels.py:54-122) on the GPU, in place."""
    CALLS["forward_kernel"] += 1
    import torch

    B, T, D = expl.shape
    G, S = final_probs.shape
    I = bw_from.shape[1]

    def build():
        n_arcs = bw_index[:, :, 1].max(axis=1).astype(np.int64) if S else np.zeros(G, np.int64)
        bw_to = _from_ranges(bw_index, n_arcs, I)
        # forward_* (by source) order is only needed for the handle; derive it stably.
        fw = [np.zeros((G, I), np.uint32), np.zeros((G, I), np.uint32),
              np.zeros((G, I), np.uint32), np.zeros((G, I), np.float64)]
        for g in range(G):
            n = int(n_arcs[g])
            o = np.argsort(bw_from[g, :n], kind="stable")
            fw[0][g, :n] = bw_from[g, :n][o]
            fw[1][g, :n] = bw_to[g, :n][o]
            fw[2][g, :n] = bw_pdf[g, :n][o]
            fw[3][g, :n] = bw_prob[g, :n][o]
        return _create(G, S, I, D, n_arcs, fw, (bw_from, bw_to, bw_pdf, bw_prob), final_probs,
                       init_states)

    h = _graph_handle("fwd", (bw_from, bw_pdf, bw_prob, bw_index, final_probs), build)
    d_expl = _dev(expl, torch.float64)
    d_len = _dev(lengths, torch.int32)
    d_rm = _dev(row_map, torch.int64)
    d_pi = _dev(leak_pi, torch.float64)
    d_alpha = _dev(alpha, torch.float64)
    d_scales = _dev(scales, torch.float64)
    d_fail = _dev(fail_frames, torch.int64)
    _check(library().lfmmi_forward_kernel(
        h, d_rm.data_ptr(), B, T, D, d_expl.data_ptr(), d_len.data_ptr(), float(leak),
        d_pi.data_ptr(), float(scale_floor), d_alpha.data_ptr(), d_scales.data_ptr(),
        d_fail.data_ptr(), _stream()))
    _copy_back(alpha, d_alpha)
    _copy_back(scales, d_scales)
    _copy_back(fail_frames, d_fail)


def backward_kernel(expl, lengths, bvalid, row_map, fw_to, fw_pdf, fw_prob, fw_index,
                    final_probs, scales, leak, leak_pi, fail_frames, beta):
    """``_kernels.backward_kernel`` (_kernels.py:125-191) on the GPU, in place."""
    CALLS["backward_kernel"] += 1
    import torch

    B, T, D = expl.shape
    G, S = final_probs.shape
    I = fw_to.shape[1]

    def build():
        n_arcs = fw_index[:, :, 1].max(axis=1).astype(np.int64) if S else np.zeros(G, np.int64)
        fw_from = _from_ranges(fw_index, n_arcs, I)
        return _create(G, S, I, D, n_arcs, (fw_from, fw_to, fw_pdf, fw_prob), None, final_probs,
                       np.zeros(G, np.uint32))

    h = _graph_handle("bwd", (fw_to, fw_pdf, fw_prob, fw_index, final_probs), build)
    d_expl = _dev(expl, torch.float64)
    d_len = _dev(lengths, torch.int32)
    d_rm = _dev(row_map, torch.int64)
    d_sc = _dev(scales, torch.float64)
    d_pi = _dev(leak_pi, torch.float64)
    d_fail = _dev(fail_frames, torch.int64)
    d_beta = _dev(beta, torch.float64)
    _check(library().lfmmi_backward_kernel(
        h, d_rm.data_ptr(), B, T, D, d_expl.data_ptr(), d_len.data_ptr(), d_sc.data_ptr(),
        float(leak), d_pi.data_ptr(), d_fail.data_ptr(), d_beta.data_ptr(), _stream()))
    _copy_back(beta, d_beta)


def posterior_kernel(expl, lengths, row_map, item_ntrans, fw_from, fw_to, fw_pdf, fw_prob,
                     alpha, beta, fail_frames, gamma):
    """``_kernels.posterior_kernel`` (_kernels.py:194-224) on the GPU, in place."""
    CALLS["posterior_kernel"] += 1
    import torch

    B, T, D = expl.shape
    G, I = fw_from.shape
    S = alpha.shape[2]

    def build():
        n_arcs = np.zeros(G, np.int64)
        rm = np.asarray(row_map, np.int64)
        n_arcs[rm] = np.asarray(item_ntrans, np.int64)
        return _create(G, S, I, D, n_arcs, (fw_from, fw_to, fw_pdf, fw_prob), None,
                       np.zeros((G, S)), np.zeros(G, np.uint32))

    h = _graph_handle("post", (fw_from, fw_to, fw_pdf, fw_prob, item_ntrans), build)
    d_expl = _dev(expl, torch.float64)
    d_len = _dev(lengths, torch.int32)
    d_rm = _dev(row_map, torch.int64)
    d_alpha = _dev(alpha, torch.float64)
    d_beta = _dev(beta, torch.float64)
    d_fail = _dev(fail_frames, torch.int64)
    d_gamma = _dev(gamma, torch.float64)
    _check(library().lfmmi_posterior_kernel(
        h, d_rm.data_ptr(), B, T, D, d_expl.data_ptr(), d_len.data_ptr(), d_alpha.data_ptr(),
        d_beta.data_ptr(), d_fail.data_ptr(), d_gamma.data_ptr(), _stream()))
    _copy_back(gamma, d_gamma)


def install(chainloss_module) -> None:
    """Rebind ``chainloss._kernels.{forward,backward,posterior}_kernel`` to the GPU seam."""
    k = chainloss_module._kernels
    _SAVED[id(k)] = (k.forward_kernel, k.backward_kernel, k.posterior_kernel)
    k.forward_kernel = forward_kernel
    k.backward_kernel = backward_kernel
    k.posterior_kernel = posterior_kernel


def uninstall(chainloss_module) -> None:
    k = chainloss_module._kernels
    saved = _SAVED.pop(id(k), None)
    if saved:
        k.forward_kernel, k.backward_kernel, k.posterior_kernel = saved
