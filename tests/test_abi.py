"""CPU checks of the boundary: libgps.so (built for sm_100a) loads without a GPU, exports every
function include/gps.h declares, and its binding declares the same set.  No compute calls."""
import ctypes
import subprocess

import pytest

from paper_2509_11574_b200 import _native as N


def test_header_declares_the_four_hot_calls():
    syms = N.declared_symbols()
    for s in ("gps_fuse", "gps_raycast", "gps_render", "gps_refine_step"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    lib = N.load()
    for s in N.declared_symbols():
        assert hasattr(lib, s), s
    assert set(N.PROTOTYPES) == set(N.declared_symbols())
    assert lib.gps_abi_version() == 4
    assert lib.gps_status_string(2) == b"GPS_ERR_OUT_OF_BLOCKS"


def test_library_is_sm100a_code():
    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_argument_validation_is_synchronous_and_needs_no_gpu():
    lib = N.load()
    cfg = N.gps_volume_config(0.005, 0.02, 300, 0.1, 10.0, 16, 1000)  # w_max > 255, slots not 2^k
    h = ctypes.c_void_p()
    assert lib.gps_volume_create(ctypes.byref(cfg), None, ctypes.byref(h)) == 1
    assert b"bad config" in lib.gps_last_error()
    rc = N.gps_render_config(0.02, 1 / 255, 0.2, 0.3, 12, 0, 0, 0, 0)  # tile must be 8 or 16
    K = N.gps_intrinsics(60, 60, 31.5, 23.5, 64, 48)
    assert lib.gps_render_workspace_size(10, ctypes.byref(K), ctypes.byref(rc)) == 0
    rc.tile = 16
    assert lib.gps_render_workspace_size(10, ctypes.byref(K), ctypes.byref(rc)) > 0


def test_colour_mean_magic_division_is_exact():
    """k_integrate divides the colour running-mean numerator (<= 255*255 + 255 + 128) by w+1
    (1..256) as a multiply-high by ceil(2^32/(w+1)); exhaustively equal to integer division, so
    the colour stays bit-exact with the oracle's plain division (R-INT)."""
    import numpy as np
    n = np.arange(0, 255 * 255 + 255 + 129, dtype=np.uint64)
    for d in range(2, 257):  # d = w + 1; w = 0 copies the sample instead (M would be 2^32)
        M32 = np.uint32((np.uint32(0xFFFFFFFF) // np.uint32(d)) + np.uint32(1))  # u32 as on device
        assert int(M32) == -(-(1 << 32) // d)
        assert np.array_equal((n * np.uint64(M32)) >> np.uint64(32), n // np.uint64(d)), d


def test_footprint_walk_division_is_exact():
    """k_backward maps lane index k < 256 of a w <= 16 wide footprint to (k / w, k % w) with
    (k * ceil(2^16 / w)) >> 16; exhaustively exact."""
    for w in range(1, 17):
        magic = (65536 + w - 1) // w
        for k in range(256):
            assert (k * magic) >> 16 == k // w, (w, k)


def test_refine_round_rejects_uneven_view_lists_before_any_launch():
    """The binding checks the round's per-iteration view lists (all the same length) on the host,
    before it builds any argument for the library."""
    from paper_2509_11574_b200 import api as A
    ras = A.Rasterizer.__new__(A.Rasterizer)  # no workspace: the check comes first
    with pytest.raises(ValueError):
        ras.refine_round(None, None, [], [[0], [0, 1]])


def test_graph_entry_points_are_declared():
    syms = N.declared_symbols()
    assert "gps_refine_round" in syms and "gps_fuse_raycast" in syms
