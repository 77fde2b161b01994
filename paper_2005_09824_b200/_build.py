"""In-tree build of the native pieces (run by ``__graft_entry__.build()``).

1. ``_lib/libpaper_lfmmi.so`` — the C-ABI library (``include/lfmmi.h``):
   CUDA kernels + host graph packer, compiled by nvcc for sm_100a only.
2. ``_lib/_lfmmi_torch.so`` — the PyTorch C++ extension (tensor/stream
   plumbing), linked against (1) with an ``$ORIGIN`` rpath.

Both land inside the package directory so they travel with the repo snapshot
to the GPU box; nothing is cached under ``~/.cache``.
"""

from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
# Build-time variants for same-box A/B measurements (development only): an
# extra set of -D flags, built into _lib_<name>/ and selected at import time
# by LFMMI_LIB_VARIANT=<name>.  The default build is _lib/.
VARIANTS = {"rows8": ["-DLFMMI_SLOT_ROWS=8"], "l2r12": ["-DLFMMI_L2_ROWS=12"],
            "l2r16": ["-DLFMMI_L2_ROWS=16"]}
VARIANT = os.environ.get("LFMMI_LIB_VARIANT", "")
LIB_DIR = os.path.join(PKG, "_lib" + (f"_{VARIANT}" if VARIANT else ""))
CORE_SO = os.path.join(LIB_DIR, "libpaper_lfmmi.so")
TORCH_SO = os.path.join(LIB_DIR, "_lfmmi_torch" + (sysconfig.get_config_var("EXT_SUFFIX") or ".so"))

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CORE_SOURCES = ["lfmmi_api.cu", "lfmmi_group.cu", "lfmmi_tile.cu", "lfmmi_linear.cu", "lfmmi_stream.cu", "lfmmi_streamsplit.cu", "lfmmi_split.cu",
                "lfmmi_graph.cpp",
                "lfmmi_schedule.cpp", "lfmmi_fst.cpp", "lfmmi_options.cpp"]


def _run(cmd, verbose):
    if verbose:
        print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build_core(verbose=True, force=False):
    srcs = [os.path.join(CSRC, s) for s in CORE_SOURCES]
    deps = srcs + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    deps.append(os.path.join(INCLUDE, "lfmmi.h"))
    if not force and not _stale(CORE_SO, deps):
        return CORE_SO
    os.makedirs(LIB_DIR, exist_ok=True)
    objs = [os.path.join(LIB_DIR, os.path.basename(s) + ".o") for s in srcs]
    cmds = [[NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
             "-Xptxas", "-v" if os.environ.get("LFMMI_PTXAS_VERBOSE") else "-O3",
             *VARIANTS.get(VARIANT, []),
             "-x", "cu" if s.endswith(".cu") else "c++",
             "-I", INCLUDE, "-I", CSRC, "-c", s, "-o", o] for s, o in zip(srcs, objs)]
    # translation units are independent: compile them concurrently
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 1)) as pool:
        for f in [pool.submit(_run, c, verbose) for c in cmds]:
            f.result()
    _run([NVCC, *ARCH, "-shared", "-o", CORE_SO, *objs, "-lcudart"], verbose)
    for o in objs:
        os.remove(o)
    return CORE_SO


def build_torch_ext(verbose=True, force=False):
    import torch
    from torch.utils import cpp_extension

    src = os.path.join(CSRC, "torch_ext.cpp")
    if not force and not _stale(TORCH_SO, [src, CORE_SO, os.path.join(INCLUDE, "lfmmi.h")]):
        return TORCH_SO
    incs = cpp_extension.include_paths(device_type="cuda") + [INCLUDE, sysconfig.get_paths()["include"]]
    abi = int(torch._C._GLIBCXX_USE_CXX11_ABI)
    cmd = ["g++", "-O2", "-fPIC", "-shared", "-std=c++17",
           f"-D_GLIBCXX_USE_CXX11_ABI={abi}", "-DTORCH_EXTENSION_NAME=_lfmmi_torch",
           "-DTORCH_API_INCLUDE_EXTENSION_H",
           *[f"-I{p}" for p in incs], src, "-o", TORCH_SO,
           f"-L{LIB_DIR}", "-lpaper_lfmmi", "-Wl,-rpath,$ORIGIN",
           *[f"-L{p}" for p in cpp_extension.library_paths(device_type="cuda")],
           "-lc10", "-lc10_cuda", "-ltorch", "-ltorch_cpu", "-ltorch_cuda", "-ltorch_python",
           "-lcudart"]
    _run(cmd, verbose)
    return TORCH_SO


def build_all(verbose=True, force=False):
    build_core(verbose, force)
    build_torch_ext(verbose, force)


if __name__ == "__main__":
    build_all(verbose=True, force="--force" in sys.argv)
