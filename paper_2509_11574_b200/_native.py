"""ctypes mirror of include/gps.h (argument marshalling only).

Every step of the mapping path runs in libgps.so's CUDA kernels; this module only declares the
C structs and function prototypes.  There is no fallback: if libgps.so is missing or cannot be
loaded, importing the API raises.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgps.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "gps.h")

gps_stream_t = C.c_void_p
gps_status = C.c_int

STATUS = {0: "GPS_OK", 1: "GPS_ERR_INVALID_ARG", 2: "GPS_ERR_OUT_OF_BLOCKS",
          3: "GPS_ERR_WORKSPACE_TOO_SMALL", 4: "GPS_ERR_CUDA", 5: "GPS_ERR_OOM"}


class gps_intrinsics(C.Structure):
    _fields_ = [("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("width", C.c_int32), ("height", C.c_int32)]


class gps_pose(C.Structure):
    _fields_ = [("R", C.c_float * 9), ("t", C.c_float * 3)]


class gps_volume_config(C.Structure):
    _fields_ = [("voxel_size", C.c_float), ("mu", C.c_float), ("w_max", C.c_int32),
                ("depth_min", C.c_float), ("depth_max", C.c_float), ("max_blocks", C.c_int64),
                ("hash_slots", C.c_int64), ("dense_origin", C.c_int32 * 3), ("dense_dims", C.c_int32 * 3)]


class gps_gaussians(C.Structure):
    _fields_ = [("n", C.c_int64), ("sh_degree", C.c_int32), ("xyz", C.c_void_p),
                ("log_scale", C.c_void_p), ("rot", C.c_void_p), ("opacity_raw", C.c_void_p),
                ("sh", C.c_void_p)]


class gps_render_config(C.Structure):
    _fields_ = [("eps_depth", C.c_float), ("alpha_min", C.c_float), ("near_z", C.c_float),
                ("lowpass", C.c_float), ("tile", C.c_int32), ("tile_depth_precull", C.c_int32),
                ("max_pairs", C.c_int64), ("sort_free", C.c_int32), ("backward", C.c_int32)]


class gps_adam_config(C.Structure):
    _fields_ = [("lr_xyz", C.c_float), ("lr_sh0", C.c_float), ("lr_shrest", C.c_float),
                ("lr_opacity", C.c_float), ("lr_scale", C.c_float), ("lr_rot", C.c_float),
                ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float)]


class gps_adam_state(C.Structure):
    _fields_ = [("m", gps_gaussians), ("v", gps_gaussians), ("step", C.c_int64)]


class gps_view(C.Structure):
    _fields_ = [("K", gps_intrinsics), ("T", gps_pose), ("sdf_depth", C.c_void_p),
                ("sdf_color", C.c_void_p), ("target_rgba", C.c_void_p)]


class gps_add_config(C.Structure):
    _fields_ = [("delta_c", C.c_float), ("delta_w", C.c_float), ("sample_frac", C.c_float),
                ("opacity_init", C.c_float), ("scale_max", C.c_float), ("knn_cell", C.c_float),
                ("seed", C.c_uint32), ("reserved", C.c_int32)]


class gps_remove_config(C.Structure):
    _fields_ = [("sigma_min", C.c_float), ("scale_max", C.c_float), ("scale_min", C.c_float),
                ("reserved", C.c_int32)]


class gps_icp_config(C.Structure):
    _fields_ = [("levels", C.c_int32), ("iters", C.c_int32 * 4), ("dist_max", C.c_float),
                ("angle_max_deg", C.c_float), ("depth_min", C.c_float), ("depth_max", C.c_float),
                ("eps", C.c_float), ("min_inlier_frac", C.c_float), ("fallback", C.c_int32), ("min_inlier_px_frac", C.c_float), ("min_pivot_ratio", C.c_float),
                ("filter_radius", C.c_int32), ("filter_sigma_s", C.c_float), ("filter_sigma_r", C.c_float)]


class gps_track_result(C.Structure):
    _fields_ = [("T", gps_pose), ("R64", C.c_double * 9), ("t64", C.c_double * 3), ("energy", C.c_double),
                ("inliers", C.c_int32), ("valid", C.c_int32), ("steps", C.c_int32), ("degenerate", C.c_int32),
                ("converged", C.c_int32), ("inlier_frac", C.c_float), ("pivot_ratio", C.c_float),
                ("reserved", C.c_int32)]


P = C.POINTER
vp, i64, i32, f32, sz = C.c_void_p, C.c_int64, C.c_int32, C.c_float, C.c_size_t

PROTOTYPES = {
    "gps_volume_create": (gps_status, [P(gps_volume_config), gps_stream_t, P(vp)]),
    "gps_volume_destroy": (None, [vp]),
    "gps_volume_reset": (gps_status, [vp, gps_stream_t]),
    "gps_volume_copy": (gps_status, [vp, vp, gps_stream_t]),
    "gps_volume_stats_sync": (gps_status, [vp, gps_stream_t, P(i64), P(i64), P(i64), P(i64), P(i64)]),
    "gps_fuse": (gps_status, [vp, P(gps_intrinsics), P(gps_pose), vp, f32, vp, gps_stream_t]),
    "gps_raycast": (gps_status, [vp, P(gps_intrinsics), P(gps_pose), vp, vp, vp, gps_stream_t]),
    "gps_fuse_raycast": (gps_status, [vp, P(gps_intrinsics), P(gps_pose), vp, f32, vp, vp, vp, vp, i32,
                                      gps_stream_t]),
    "gps_fuse_dpose": (gps_status, [vp, P(gps_intrinsics), vp, vp, f32, vp, gps_stream_t]),
    "gps_raycast_dpose": (gps_status, [vp, P(gps_intrinsics), vp, vp, vp, vp, gps_stream_t]),
    "gps_render_workspace_size": (sz, [i64, P(gps_intrinsics), P(gps_render_config)]),
    "gps_render": (gps_status, [P(gps_gaussians), P(gps_intrinsics), P(gps_pose), vp, vp, vp,
                                P(gps_render_config), vp, sz, vp, vp, vp, gps_stream_t]),
    "gps_refine_workspace_size": (sz, [i64, P(gps_intrinsics), P(gps_render_config), i32]),
    "gps_refine_step": (gps_status, [P(gps_gaussians), P(gps_adam_state), P(gps_view), i32,
                                     P(gps_render_config), P(gps_adam_config), vp, sz, vp,
                                     P(gps_gaussians), gps_stream_t]),
    "gps_refine_round": (gps_status, [P(gps_gaussians), P(gps_adam_state), P(gps_view), i32, P(i32), i32, i32,
                                      P(gps_render_config), P(gps_adam_config), vp, sz, vp, i32, gps_stream_t]),
    "gps_adam_step": (gps_status, [P(gps_gaussians), P(gps_adam_state), P(gps_gaussians),
                                   P(gps_adam_config), gps_stream_t]),
    "gps_render_stats_sync": (gps_status, [vp, gps_stream_t, P(i64), P(i64), P(i64)]),
    "gps_vertex_normals": (gps_status, [P(gps_intrinsics), P(gps_pose), vp, vp, vp, gps_stream_t]),
    "gps_vertex_normals_dpose": (gps_status, [P(gps_intrinsics), vp, vp, vp, vp, gps_stream_t]),
    "gps_add_workspace_size": (sz, [P(gps_intrinsics)]),
    "gps_add_gaussians_sync": (gps_status, [P(gps_gaussians), i64, P(gps_adam_state), P(gps_intrinsics), vp, vp,
                                            vp, vp, vp, vp, P(gps_add_config), vp, sz, P(i64), P(i64),
                                            gps_stream_t]),
    "gps_remove_workspace_size": (sz, [i64, i32]),
    "gps_track_workspace_size": (sz, [P(gps_intrinsics), i32]),
    "gps_track_sync": (gps_status, [P(gps_intrinsics), vp, f32, vp, vp, P(gps_pose), P(gps_pose), P(gps_icp_config),
                                    vp, sz, P(gps_track_result), gps_stream_t]),
    "gps_pose_extrapolate": (gps_status, [vp, vp, vp, gps_stream_t]),
    "gps_track_async": (gps_status, [P(gps_intrinsics), vp, f32, vp, vp, vp, vp, vp, P(gps_icp_config), vp, sz, vp,
                                     vp, gps_stream_t]),
    "gps_remove_gaussians_sync": (gps_status, [P(gps_gaussians), P(gps_adam_state), P(gps_remove_config), vp, sz,
                                               P(i64), gps_stream_t]),
    "gps_debug_export_blocks_sync": (gps_status, [vp, gps_stream_t, vp, vp, i64, P(i64)]),
    "gps_debug_export_visible_sync": (gps_status, [vp, gps_stream_t, vp, i64, P(i64)]),
    "gps_debug_apron_check_sync": (gps_status, [vp, gps_stream_t, P(i64)]),
    "gps_debug_hash_check_sync": (gps_status, [vp, gps_stream_t, P(i64)]),
    "gps_debug_check_word_sync": (gps_status, [P(i64), P(C.c_int32)]),
    "gps_debug_check_selftest": (gps_status, [C.c_int32, gps_stream_t]),
    "gps_debug_raycast_footprint_sync": (gps_status, [vp, P(gps_intrinsics), P(gps_pose), gps_stream_t, P(i64)]),
    "gps_debug_render_lists_sync": (gps_status, [vp, gps_stream_t, vp, i64, vp, P(i64)]),
    "gps_debug_render_counts_sync": (gps_status, [P(gps_gaussians), P(gps_intrinsics), P(gps_pose), vp, vp,
                                                  P(gps_render_config), vp, sz, P(i64), P(i64), gps_stream_t]),
    "gps_profile_enable": (None, [C.c_int]),
    "gps_profile_read_sync": (C.c_int, [C.c_char_p, C.c_int, P(C.c_double), P(i64), C.c_int]),
    "gps_profile_timeline_sync": (i64, [P(C.c_int32), P(C.c_double), P(C.c_double), i64]),
    "gps_status_string": (C.c_char_p, [gps_status]),
    "gps_last_error": (C.c_char_p, []),
    "gps_abi_version": (C.c_int, []),
}


def declared_symbols() -> list[str]:
    """Every function include/gps.h declares (parsed from the header)."""
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(gps_[a-z0-9_]+)\s*\(", txt)))


_lib = None


class GPSError(RuntimeError):
    def __init__(self, fn: str, status: int, msg: str):
        super().__init__(f"{fn} -> {STATUS.get(status, status)}: {msg}")
        self.status = status


def load(path: str | None = None):
    """Load libgps.so (raises OSError if it is missing: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    p = path or os.environ.get("GPS_LIB") or LIB_PATH  # GPS_LIB: A/B builds (tools/ab.sh) only
    if not os.path.exists(p):
        raise OSError(f"libgps.so not built at {p}: run `python paper_2509_11574_b200/build.py`")
    L = C.CDLL(p)
    for name, (res, args) in PROTOTYPES.items():
        if name.startswith("gps_debug_") and not hasattr(L, name):
            continue  # an older A/B build without a later debug hook
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    if L.gps_abi_version() != ABI_VERSION:
        raise OSError(f"libgps.so ABI {L.gps_abi_version()} != binding ABI {ABI_VERSION}: rebuild")
    _lib = L
    return L


ABI_VERSION = 4  # must equal GPS_ABI_VERSION of include/gps.h (the struct layouts above)


def check(fn: str, status: int):
    if status != 0:
        msg = _lib.gps_last_error().decode() if _lib is not None else ""
        raise GPSError(fn, status, msg)
