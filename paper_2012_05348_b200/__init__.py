"""B200-native batched compressed-BVH collision detection and proximity query
(arXiv 2012.05348).  See DESIGN.md; the C-ABI is include/cbvh.h."""
from .api import (CompressedBVH, Workspace, blob_info, build_compressed_bvh, check,  # noqa: F401
                  collide_batch, distance_batch, last_launch_count, read_stats,
                  validate_poses)
