"""B200-native (sm_100a) Gaussian-Plus-SDF mapping step of GPS-SLAM (arXiv 2509.11574).

The compute path is libgps.so (hand-written CUDA behind the C ABI of include/gps.h); this
package is the thin Python binding (``api``), the host-side round schedule (``schedule``) and
the in-tree build (``build``).  Importing it loads libgps.so and raises if it is missing.
"""
from . import _native
from .api import (AdamConfig, AdamState, AddConfig, Camera, Gaussians, Rasterizer, RemoveConfig, RenderConfig, View,
                  Volume, adam_step, add_gaussians, pose_struct, remove_gaussians, vertex_normals, IcpConfig, track,
                  TRACK_RESULT_BYTES, pose_extrapolate, pose_tensor, track_async, track_result, vertex_normals_dpose)

__all__ = ["AdamConfig", "AdamState", "AddConfig", "Camera", "Gaussians", "Rasterizer", "RemoveConfig", "RenderConfig",
           "View", "Volume", "adam_step", "add_gaussians", "pose_struct", "remove_gaussians", "vertex_normals",
           "IcpConfig", "track", "TRACK_RESULT_BYTES", "pose_extrapolate", "pose_tensor", "track_async", "track_result",
           "vertex_normals_dpose"]
