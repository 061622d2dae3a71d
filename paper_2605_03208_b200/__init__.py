"""paper_2605_03208_b200 -- B200-native (sm_100a) hot path of Kerncap's
capture-and-validate loop (arXiv 2605.03208): the address-space closure.

The product is ``libkc.so`` (hand-written CUDA kernels + C ABI, include/kc.h);
:mod:`paper_2605_03208_b200.kc` is its thin ctypes binding and
:mod:`paper_2605_03208_b200.dist` the multi-GPU combine over torch.distributed.
"""
from . import kc  # noqa: F401

__all__ = ["kc"]
