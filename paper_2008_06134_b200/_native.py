"""ctypes binding of the sbrc C ABI (include/sbrc.h).

The shared library ``_sbrc.so`` is built in-tree by ``build.py`` (nvcc,
``-gencode arch=compute_100a,code=sm_100a``). There is no fallback: if the
library is missing this module raises ImportError at import time, and every
call checks the returned status.
"""

from __future__ import annotations

import ctypes as C
import os

from .scene import ConfigError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SBRC_LIB") or os.path.join(_HERE, "_sbrc.so")  # SBRC_LIB: A/B experiments

ABI_VERSION = 12
MAX_SHELLS = 8
MAX_ANGLES = 16
MAX_PEERS = 8
MAX_CLIP = 4

OK, EINVAL, ECONFIG, ECUDA, EUNSUPPORTED = 0, -1, -2, -3, -4
VOXEL_F32, VOXEL_U8, VOXEL_U16 = 0, 1, 2
SHADE = {"none": 0, "sbrc_shadow": 1, "shell": 2, "cone": 3, "phong": 4, "extinction": 5}
LOOKUP = {"linear": 0, "nearest": 1}

#: every symbol include/sbrc.h declares
EXPORTS = ("sbrc_abi_version", "sbrc_strerror", "sbrc_struct_size", "sbrc_volume_check",
           "sbrc_build", "sbrc_render", "sbrc_pack_quads", "sbrc_shadow_oracle", "sbrc_light_factor",
           "sbrc_normalize_f32", "sbrc_half_angle", "sbrc_ipc_alloc", "sbrc_ipc_free", "sbrc_ipc_handle",
           "sbrc_ipc_open", "sbrc_ipc_close", "sbrc_march_grid", "sbrc_local_rows",
           "sbrc_render_grid", "sbrc_host_device_pointer", "sbrc_debug_violations", "sbrc_widen_volume",
           "sbrc_tile_order", "sbrc_permute_rows", "sbrc_volume_layout", "sbrc_brick_elems", "sbrc_brick_pack")

D3 = C.c_double * 3
D2 = C.c_double * 2


class SbrcVolume(C.Structure):
    _fields_ = [("data", C.c_void_p), ("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32),
                ("voxel_type", C.c_int32), ("box_lo", D3), ("box_ext", D3)]


class SbrcLightFrame(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("n_slices", C.c_int32),
                ("_pad", C.c_int32), ("axis_u", D3), ("axis_v", D3), ("light_dir", D3),
                ("u_range", D2), ("v_range", D2), ("d_min", C.c_double), ("d_max", C.c_double),
                ("plane_offsets", C.c_void_p)]


class SbrcBuildParams(C.Structure):
    _fields_ = [("volume", SbrcVolume), ("light", SbrcLightFrame), ("alpha_lut", C.c_void_p),
                ("compensation_n", C.c_double), ("row_begin", C.c_int32), ("row_end", C.c_int32),
                ("quads", C.c_void_p), ("quad_layer_stride", C.c_int64), ("quad_row_stride", C.c_int64),
                ("write_reach", C.c_double), ("write_below", C.c_int32), ("write_above", C.c_int32),
                ("write_sparse", C.c_int32), ("output_plain", C.c_int32),
                ("n_clip", C.c_int32), ("clip", (C.c_double * 4) * MAX_CLIP), ("quad_layout", C.c_int32)]


class SbrcRenderParams(C.Structure):
    _fields_ = [("volume", SbrcVolume), ("lut_rgba", C.c_void_p),
                ("width", C.c_int32), ("height", C.c_int32), ("shading", C.c_int32), ("lookup", C.c_int32),
                ("eye", D3), ("forward", D3), ("right", D3), ("up2", D3),
                ("tan_half", C.c_double), ("aspect", C.c_double), ("step", C.c_double),
                ("et_alpha", C.c_double), ("light", SbrcLightFrame), ("quads", C.c_void_p),
                ("quad_layer_stride", C.c_int64), ("quad_row_stride", C.c_int64),
                ("light_color", C.c_float * 3), ("ambient_floor", C.c_float),
                ("shell_count", C.c_int32), ("cone_axis_samples", C.c_int32),
                ("cone_angle_count", C.c_int32), ("skip_clear", C.c_int32),
                ("shell_radius", C.c_double * MAX_SHELLS), ("shell_weight", C.c_double * MAX_SHELLS),
                ("cone_ring", C.c_double), ("cone_cos", C.c_double * MAX_ANGLES),
                ("cone_sin", C.c_double * MAX_ANGLES),
                ("band_rows", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32), ("local_rows", C.c_int32),
                ("scene_light_dir", D3), ("phong", C.c_double * 4), ("voxel_size", D3),
                ("image", C.c_void_p), ("peer_images", C.c_void_p * MAX_PEERS), ("n_peers", C.c_int32),
                ("n_tiles", C.c_int32), ("tile_order", C.c_void_p), ("sample_count", C.c_void_p),
                ("tile_steps", C.c_void_p), ("row_begin", C.c_int32), ("row_count", C.c_int32),
                ("march_kernel", C.c_int32), ("quad_layout", C.c_int32)]


class SbrcHalfAngleParams(C.Structure):
    _fields_ = [("volume", SbrcVolume), ("lut", C.c_void_p), ("plane_offsets", C.c_void_p),
                ("width", C.c_int32), ("height", C.c_int32), ("light_width", C.c_int32),
                ("light_height", C.c_int32), ("n_slices", C.c_int32), ("front_to_back", C.c_int32),
                ("eye", D3), ("forward", D3), ("right", D3), ("up2", D3), ("tan_half", C.c_double),
                ("aspect", C.c_double), ("half", D3), ("delta", C.c_double), ("light_dir", D3), ("axis_u", D3),
                ("axis_v", D3), ("u_range", D2), ("v_range", D2), ("hl", C.c_double), ("h_dot_u", C.c_double),
                ("h_dot_v", C.c_double), ("h_dot_e", C.c_double), ("eye_accum", C.c_void_p),
                ("light_accum", C.c_void_p), ("image", C.c_void_p)]


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"sbrc CUDA library not built: {LIB_PATH} is missing "
            "(run `python paper_2008_06134_b200/build.py` or __graft_entry__.build())")
    lib = C.CDLL(LIB_PATH)
    lib.sbrc_abi_version.restype = C.c_int
    lib.sbrc_strerror.restype = C.c_char_p
    lib.sbrc_strerror.argtypes = [C.c_int]
    lib.sbrc_struct_size.restype = C.c_int64
    lib.sbrc_struct_size.argtypes = [C.c_int]
    lib.sbrc_volume_check.argtypes = [C.POINTER(SbrcVolume)]
    lib.sbrc_build.argtypes = [C.POINTER(SbrcBuildParams), C.c_void_p]
    lib.sbrc_render.argtypes = [C.POINTER(SbrcRenderParams), C.c_void_p]
    lib.sbrc_local_rows.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int]
    lib.sbrc_march_grid.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int * 4]
    lib.sbrc_render_grid.argtypes = [C.POINTER(SbrcRenderParams), C.c_int * 4]
    lib.sbrc_light_factor.argtypes = [C.POINTER(SbrcRenderParams), C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                      C.c_void_p]
    lib.sbrc_ipc_alloc.argtypes = [C.c_int64, C.POINTER(C.c_void_p)]
    lib.sbrc_ipc_free.argtypes = [C.c_void_p]
    lib.sbrc_host_device_pointer.argtypes = [C.c_void_p, C.POINTER(C.c_void_p)]
    lib.sbrc_ipc_handle.argtypes = [C.c_void_p, C.c_char * 64]
    lib.sbrc_ipc_open.argtypes = [C.c_char * 64, C.POINTER(C.c_void_p)]
    lib.sbrc_ipc_close.argtypes = [C.c_void_p]
    lib.sbrc_half_angle.argtypes = [C.POINTER(SbrcHalfAngleParams), C.c_int, C.c_int, C.c_int, C.c_int,
                                    C.POINTER(C.c_int), C.c_void_p]
    lib.sbrc_debug_violations.argtypes = [C.POINTER(C.c_uint * 8), C.c_int]
    lib.sbrc_normalize_f32.argtypes = [C.c_void_p, C.c_int64, C.c_float, C.c_float, C.c_void_p]
    lib.sbrc_widen_volume.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_void_p]
    lib.sbrc_tile_order.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
    lib.sbrc_volume_layout.restype = C.c_int
    lib.sbrc_brick_elems.argtypes = [C.c_int, C.c_int, C.c_int]
    lib.sbrc_brick_elems.restype = C.c_int64
    lib.sbrc_brick_pack.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
    lib.sbrc_permute_rows.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p]
    lib.sbrc_shadow_oracle.argtypes = [C.POINTER(SbrcVolume), C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                       C.c_double, C.c_void_p, C.c_void_p]
    lib.sbrc_pack_quads.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int,
                                    C.c_void_p, C.c_int64, C.c_int64, C.c_void_p]
    if lib.sbrc_abi_version() != ABI_VERSION:
        raise ImportError(f"sbrc ABI mismatch: library {lib.sbrc_abi_version()} != binding {ABI_VERSION}")
    sizes = (SbrcVolume, SbrcLightFrame, SbrcBuildParams, SbrcRenderParams, SbrcHalfAngleParams)
    for i, st in enumerate(sizes):
        if lib.sbrc_struct_size(i) != C.sizeof(st):
            raise ImportError(f"sbrc struct {st.__name__} layout mismatch: "
                              f"C {lib.sbrc_struct_size(i)} vs ctypes {C.sizeof(st)}")
    return lib


lib = _load()


def check(status: int, what: str) -> None:
    """Map a C status to the reference's exception types."""
    if status == OK:
        return
    msg = f"{what}: {lib.sbrc_strerror(status).decode()}"
    if status == ECONFIG:
        raise ConfigError(msg)
    if status in (EINVAL, EUNSUPPORTED):
        raise ValueError(msg)
    raise RuntimeError(msg)


def local_rows(height: int, band_rows: int, rank: int, world: int) -> int:
    return int(lib.sbrc_local_rows(height, band_rows, rank, world))


def host_device_pointer(host_ptr: int) -> int | None:
    """Device address of page-locked host memory, or None if it is not mapped."""
    d = C.c_void_p()
    if lib.sbrc_host_device_pointer(C.c_void_p(host_ptr), C.byref(d)) != OK:
        return None
    return int(d.value or 0) or None


def render_grid(p) -> tuple[int, int, int, int]:
    """(tiles_x, tiles_y, tile_w, tile_h) sbrc_render launches for params ``p``."""
    g = (C.c_int * 4)()
    check(lib.sbrc_render_grid(C.byref(p), g), "sbrc_render_grid")
    return g[0], g[1], g[2], g[3]


def march_grid(width: int, height: int, band_rows: int, rank: int, world: int) -> tuple[int, int, int, int]:
    """(tiles_x, tiles_y, tile_w, tile_h) of the throughput K2 block grid."""
    g = (C.c_int * 4)()
    check(lib.sbrc_march_grid(width, height, band_rows, rank, world, g), "sbrc_march_grid")
    return g[0], g[1], g[2], g[3]
