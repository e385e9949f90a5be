"""B200-native FlashSVD rank-aware streaming encoder (arxiv 2508.01506).

The product is the C-ABI library built from ``csrc/`` (sm_100a kernels +
C++ host runtime).  This Python package only mirrors that ABI (``abi``) and
the reference's factor containers (``model``) for tests and the bench.
"""
from . import abi  # noqa: F401

__all__ = ["abi"]
