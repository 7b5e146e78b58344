"""B200-native (sm_100a) differentiable splat rasterizer for On-the-Fly GS.

Drop-in for the reference package's operator API on the training hot path:
``render`` / ``backward`` / ``project_field`` (rasterize), ``FieldOptimizer``
(optim), ``GaussianField.densify_and_prune`` (field) and ``total_loss``
(losses).  All compute runs in hand-written CUDA kernels in ``libssr.so``
(C ABI: include/ssr.h); there is no CPU fallback.
"""

__version__ = "0.1.0"

from .camera import CameraFrame, look_at
from .errors import ExtensionMissing, InvalidParameter, NativeError, SplatError, StaleFieldError
from .field import DensifyOptions, DensifySummary, GaussianField, SparsePoint

__all__ = [
    "CameraFrame", "DensifyOptions", "DensifySummary", "ExtensionMissing", "GaussianField", "InvalidParameter",
    "NativeError", "SparsePoint", "SplatError", "StaleFieldError", "look_at", "__version__",
]
