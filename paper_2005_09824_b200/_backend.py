"""Loader for the native extension.  There is no CPU fallback: if the CUDA
extension or a GPU is missing, every compute entry point raises."""

from __future__ import annotations

import contextlib
import importlib.machinery
import importlib.util
import os

from . import _build

_EXT = None


class BackendUnavailable(RuntimeError):
    pass


def ext():
    """Import ``_lib/_lfmmi_torch`` (built in-tree by ``__graft_entry__.build``)."""
    global _EXT
    if _EXT is None:
        path = _build.TORCH_SO
        if not (os.path.exists(path) and os.path.exists(_build.CORE_SO)):
            raise BackendUnavailable(
                f"native LF-MMI extension not built ({path}); run `python -c "
                "'import __graft_entry__ as g; g.build()'` first")
        import torch  # noqa: F401  (loads libtorch before the extension)

        loader = importlib.machinery.ExtensionFileLoader("_lfmmi_torch", path)
        spec = importlib.util.spec_from_file_location("_lfmmi_torch", path, loader=loader)
        mod = importlib.util.module_from_spec(spec)
        loader.exec_module(mod)
        _EXT = mod
    return _EXT


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise BackendUnavailable("the LF-MMI hot path runs on CUDA only and no GPU is visible")
    return ext()


def core_library_path() -> str:
    return _build.CORE_SO


@contextlib.contextmanager
def options(**kw):
    """Temporarily set library options (``lfmmi_set_option``; include/lfmmi.h):
    ``with options(split=0, stream_mode="1024x1"): ...``."""
    e = ext()
    old = {k: e.get_option(k) for k in kw}
    try:
        for k, v in kw.items():
            e.set_option(k, str(v))
        yield
    finally:
        for k, v in old.items():
            e.set_option(k, v)
