"""B200-native (sm_100a) backend for the Mosaic planner hot path (arXiv 2605.18710).

The package holds only what the path needs: `csrc/` (CUDA kernels, host planner,
C ABI), `build.py`, and `mosaic.py` (Python mirror of the reference planner API).
"""
from .mosaic import *  # noqa: F401,F403
from .mosaic import Planner, load_library  # noqa: F401
