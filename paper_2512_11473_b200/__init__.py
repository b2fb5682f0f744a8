"""B200-native hot path of the contiguous sparse-grid storage of Gu & Hu
(arXiv 2512.11473): C-ABI library libsg.so (include/sg.h) with hand-written
sm_100a kernels, and its thin Python binding `sg`."""
from . import sg  # noqa: F401
from .sg import Grid, SgError  # noqa: F401
