"""pytest plugin: run the reference's own test-suite with its kernel seam bound
to this repository's CUDA kernels (tests/test_reference_suite_seam.py).

``chainloss.forward_backward`` resolves ``_kernels.{forward,backward,posterior}_kernel``
at call time (/root/reference/pkg/src/chainloss/forward_backward.py:25,187,240,273);
``kernel_seam.install`` rebinds them to ctypes wrappers of
``lfmmi_{forward,backward,posterior}_kernel`` before any test runs.
"""


def pytest_configure(config):
    import chainloss  # baseline/_ref, put first on sys.path by the caller

    from paper_2005_09824_b200 import kernel_seam

    kernel_seam.install(chainloss)
    config.lfmmi_seam = True


def pytest_unconfigure(config):
    """Record how many kernel calls went through the seam (the GPU kernels)."""
    import json
    import os

    from paper_2005_09824_b200 import kernel_seam

    path = os.environ.get("LFMMI_SEAM_REPORT")
    if path:
        with open(path, "w") as f:
            json.dump(kernel_seam.CALLS, f)


def pytest_report_header(config):
    import chainloss._kernels as k

    return f"lfmmi kernel seam: forward_kernel -> {k.forward_kernel.__module__}"
