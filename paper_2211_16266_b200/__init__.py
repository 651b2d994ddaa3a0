"""B200-native densification hot path of arxiv/paper_2211_16266 (densify360).

Equirectangular PatchMatch-Stereo for one reference keyframe over a small neighbourhood,
as hand-written sm_100a CUDA kernels behind a C ABI (include/d360.h), with the reference
package's Python entry points on top.  No CPU fallback: compute calls raise BackendError
when libd360.so or a CUDA device is missing.
"""
from .errors import BackendError, ConfigError, DatasetError, DensifyError, OrderingError
from .geometry import (
    EquirectCamera,
    GeometryError,
    PlaneHypothesis,
    RigidPose,
    camera_rays,
    pixel_to_ray,
    ray_to_pixel,
    relative_transform,
    row_latitudes,
)
from .keyframes import Keyframe, StereoGroup

__version__ = "0.1.0"

_ENGINE_NAMES = {
    "PatchSpec", "PlaneMap", "DepthPanorama", "DevicePlaneMap", "DeviceDepthPanorama", "PreparedGroup",
    "prepare_group", "random_init", "warp_plane_map", "red_black_iteration", "run_patchmatch",
    "median_outlier_filter", "to_gray", "default_top_k",
}
_PIPELINE_NAMES = {
    "ConsistencyConfig", "FusionConfig", "FusedCloud", "DepthResult", "DeviceDepthResult", "DepthStage",
    "consistency_filter", "FusionBuffer", "project_points", "POLE_LAT_LIMIT_DEG", "StreamingDensifier", "StreamOutput",
}


_INGEST_NAMES = {"resample_keyframe", "resample_image_device"}
_OFFLINE_NAMES = {"ViewFilterConfig", "ViewFilterDecision", "view_filter_accept", "KeyframeBuffer", "PipelineResult",
                  "run_offline"}


def __getattr__(name):
    # engine / pipeline import torch; keep `import paper_2211_16266_b200` light.
    if name in _ENGINE_NAMES:
        from . import engine

        return getattr(engine, name)
    if name in _PIPELINE_NAMES:
        from . import pipeline

        return getattr(pipeline, name)
    if name in _OFFLINE_NAMES:
        from . import offline

        return getattr(offline, name)
    if name in _INGEST_NAMES:
        from . import ingest

        return getattr(ingest, name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
