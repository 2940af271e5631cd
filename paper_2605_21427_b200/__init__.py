"""paper_2605_21427_b200 — B200-native hot path of the PALS / wattserve reference.

The package is the drop-in for one path: evaluating the offline
power-performance model over a dense configuration grid fused with the
constrained selection (select_config), and the batched replay of the feedback
controller (control_step). Compute runs only in libpals_gpu.so (sm_100a);
see include/pals_gpu.h for the C ABI and DESIGN.md for the design.
"""
from . import abi  # noqa: F401

__all__ = ["abi"]
