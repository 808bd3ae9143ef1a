"""B200-native distance-map pipeline: a drop-in for voxarm's map-update, EDT and
sphere-query entry points (reference: /root/reference/pkg/src/voxarm,
voxarm/__init__.py:16-37).

Every numeric result comes from hand-written sm_100a kernels in libvx.so
(csrc/); there is no CPU fallback.  Importing this package does not touch the
GPU; the library is loaded on first use and raises if it is missing.
"""

from .edt import (NO_SITE, BandConfig, DistanceField, ProximateStack, brute_force_edt,  # noqa: F401
                  default_band_config, line_nearest_sites, pba_edt, proximate_sites_1d,
                  query_nearest_site)
from .grids import (DEFAULT_HIT_LOGODDS, DEFAULT_OCCUPANCY_THRESHOLD, L_MAX, L_MIN,  # noqa: F401
                    FilterConfig, InsertStats, PointCloud, VoxelGrid, VoxelSet, load_point_cloud,
                    logit, new_grid, statistical_outlier_filter)

__all__ = [
    "NO_SITE", "BandConfig", "DistanceField", "default_band_config", "line_nearest_sites",
    "pba_edt", "query_nearest_site", "DEFAULT_HIT_LOGODDS", "DEFAULT_OCCUPANCY_THRESHOLD",
    "L_MAX", "L_MIN", "FilterConfig", "InsertStats", "PointCloud", "VoxelGrid", "VoxelSet",
    "logit", "new_grid", "ProximateStack", "brute_force_edt", "proximate_sites_1d", "load_point_cloud",
    "statistical_outlier_filter",
]
