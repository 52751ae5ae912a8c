"""B200-native deskew + live-view projections for oblique-plane stage-scan stacks.

A drop-in for the hot path of the reference ``skewstream`` package (arXiv
2211.00645): the same entry points (``ProjectionCanvas``, ``deskew_place``,
``reference_deskew``, ``warp_projection``) backed by hand-written sm_100a
kernels in ``lib/libssb.so`` (C ABI: ``include/ssb.h``), plus the additive
``deskew_volume`` (volume + fused XY/XZ/YZ max/sum projections), the pinned
multi-stream H2D pipeline (``stream``) and multi-GPU dispatch (``dist``).
"""

__version__ = "0.1.0"

from .errors import (  # noqa: F401
    CapacityError,
    DeviceError,
    EndOfStream,
    MetadataError,
    ParameterError,
    ProtocolError,
    SkewstreamError,
)
from .geometry import SheetGeometry, ViewTransform, view_transform  # noqa: F401
