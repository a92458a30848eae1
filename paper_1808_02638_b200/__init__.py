"""paper_1808_02638_b200 -- B200-native batched AMR-level advance (arXiv 1808.02638).

The compute path is ``libclaw.so`` (C-ABI, CUDA sm_100a kernels); ``binding``
is a thin ctypes layer over it.  Importing this package does not load the
library; ``binding.load()`` does, and fails loudly if it is missing.
"""
__all__ = ["binding", "workloads"]
