"""B200-native LF-MMI loss hot path (PyChain, arXiv 2005.09824).

Drop-in for the reference ``chainloss`` hot-path API
(/root/reference/pkg/src/chainloss/__init__.py:12-41): ``ChainGraph``,
``ChainGraphBatch``, ``Transition``, ``LogLikBatch``, ``make_batch``,
``unsort``, ``FBOptions``, ``forward``, ``backward``,
``occupation_posteriors``, ``forward_backward``, ``chain_loss`` — plus the
paper's torch ``ChainFunction`` / ``ChainLoss``.  All recursions run in
hand-written sm_100a CUDA behind the C-ABI in ``include/lfmmi.h``; there is
no CPU fallback.

Out of scope (not on the hot path): text-FST and PCTN file
I/O, the toy graph builder, brute-force oracle, CLI and demo trainer.
"""

from .batching import LogLikBatch, make_batch, unsort
from .forward_backward import (FBOptions, FBResult, ForwardResult, backward, forward,
                               forward_backward, forward_backward_device, get_precision,
                               occupation_posteriors, set_precision)
from .graph import ChainGraph, ChainGraphBatch, Transition, device_graphs
from .loss import (ChainFunction, ChainLoss, ChainLossResult, chain_loss, chain_loss_device,
                   chain_loss_packed)

__version__ = "0.1.0"


def set_num_threads(count: int) -> None:
    """API parity with ``chainloss.set_num_threads`` (_kernels.py:39-47).

    The GPU path has no host thread pool; the value is validated and ignored.
    """
    if count < 1:
        raise ValueError(f"thread count must be >= 1, got {count}")


def get_num_threads() -> int:
    return 1


__all__ = [
    "ChainFunction", "ChainGraph", "ChainGraphBatch", "ChainLoss", "ChainLossResult", "FBOptions",
    "FBResult", "ForwardResult", "LogLikBatch", "Transition", "backward", "chain_loss",
    "chain_loss_device", "chain_loss_packed", "device_graphs", "forward", "forward_backward",
    "forward_backward_device", "get_num_threads", "get_precision", "make_batch",
    "occupation_posteriors", "set_num_threads", "set_precision", "unsort", "__version__",
]
