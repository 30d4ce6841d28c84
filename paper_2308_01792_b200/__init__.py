"""B200-native matrix-free operator application on regularly refined
macro-tetrahedra (the hot path of arXiv 2308.01792's `blocktet`).

The product is the CUDA/C++ library libbt_b200.so behind the C ABI in
include/blocktet_b200.h; `api` mirrors the reference API over it.
"""
from .api import *  # noqa: F401,F403
from . import api  # noqa: F401
