"""B200-native (sm_100a) implementation of the NF-APACT hot path.

The product is libpact_cuda.so (include/pact_cuda.h); `api` is the Python view
of it and `include/pact/*.hpp` the C++ drop-in for the reference's pact:: API.
"""
from . import _abi  # noqa: F401

__all__ = ["_abi"]
