"""ctypes binding of the C ABI in ``include/pdg.h`` (libpdg.so, sm_100a).

The library is built in-tree by ``__graft_entry__.build()`` /
``csrc/Makefile``.  There is no fallback: if the library or a CUDA device is
missing, every entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
from functools import lru_cache

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpdg.so")

PDG_OK, PDG_ERR_INVALID, PDG_ERR_CUDA, PDG_ERR_UNSUPPORTED = 0, 1, 2, 3
ABI_VERSION = 3  # include/pdg.h PDG_ABI_VERSION
FLAG_DEGENERATE_SIMPLEX = 1 << 0
FLAG_DEGENERATE_FACET = 1 << 1
FLAG_STRADDLE = 1 << 2
FLAG_UNCLASSIFIED = 1 << 3
FLAG_NO_ADJACENT_SIMPLEX = 1 << 4
FLAG_STACK = 1 << 5
FLAG_NEG_DIFFUSION = 1 << 6
OPT_PLAIN_VOLUME = 1

MAX_CODE, MAX_CONST, MAX_STACK = 448, 96, 8
DIFF_NONE, DIFF_ISO, DIFF_FULL = 0, 1, 2
MAX_DEGREE = {2: 6, 3: 4}

_p = C.c_void_p
_i32, _i64, _f64 = C.c_int32, C.c_int64, C.c_double


class Mesh(C.Structure):
    _fields_ = [("dim", _i32),
                ("n_vertices", _i64), ("n_simplices", _i64), ("n_elements", _i64),
                ("n_faces", _i64), ("n_facets", _i64), ("n_interfaces", _i64),
                ("vertices", _p), ("simplices", _p), ("simplex_volumes", _p),
                ("elem_ptr", _p), ("elem_simplices", _p), ("elem_volumes", _p),
                ("face_owner", _p), ("face_neighbor", _p), ("face_tag", _p),
                ("face_normal", _p), ("face_measure", _p), ("face_ptr", _p),
                ("facet_vertices", _p), ("facet_owner_simplex", _p),
                ("facet_neighbor_simplex", _p), ("iface_owner", _p), ("iface_neighbor", _p),
                ("iface_ptr", _p), ("iface_faces", _p), ("elem_bface_ptr", _p),
                ("elem_bfaces", _p)]


class Basis(C.Structure):
    _fields_ = [("max_degree", _i32), ("degree", _p), ("box", _p), ("dof_offset", _p)]


class Prog(C.Structure):
    _fields_ = [("offset", _i32), ("length", _i32), ("is_const", _i32), ("pad_", _i32),
                ("value", _f64)]


class Coeffs(C.Structure):
    _fields_ = [("diffusion_kind", _i32), ("diffusion_symmetric", _i32),
                ("has_advection", _i32), ("has_reaction", _i32), ("has_source", _i32),
                ("has_dirichlet", _i32), ("has_neumann", _i32), ("pad_", _i32),
                ("diffusion", Prog * 9), ("advection", Prog * 3),
                ("reaction", Prog), ("source", Prog), ("dirichlet", Prog), ("neumann", Prog),
                ("n_code", _i32), ("n_const", _i32),
                ("code", _i32 * MAX_CODE), ("consts", _f64 * MAX_CONST)]


class Rules(C.Structure):
    _fields_ = [("max_order", _i32), ("points", _p), ("weights", _p),
                ("vol_offset", _p), ("vol_count", _p), ("face_offset", _p), ("face_count", _p),
                ("sqrt_weights", _p), ("n_points", _i32), ("pad_", _i32)]


class Params(C.Structure):
    _fields_ = [("quad_increment", _i32), ("include_gradient_terms", _i32),
                ("penalty_constant", _f64), ("coverable", _p), ("options", _i32), ("pad_", _i32)]


class Pattern(C.Structure):
    _fields_ = [("n_row_elements", _i64), ("row_elements", _p),
                ("nbr_ptr", _p), ("nbr_elem", _p), ("nbr_iface", _p),
                ("row_len", _p), ("elem_val_offset", _p), ("elem_row_offset", _p),
                ("row_ptr", _p), ("col_idx", _p), ("nbr_rec", _p), ("col_dof", _p)]


class Frames(C.Structure):
    _fields_ = [("simplex", _p), ("facet", _p), ("element", _p)]


class Slab(C.Structure):
    _fields_ = [("t0", _f64), ("t1", _f64), ("lateral_tag", _p), ("prev_values", _p),
                ("prev_dof_offset", _p), ("prev_box", _p), ("family", _i32), ("table_rows", _i32),
                ("time_rules", Rules)]


class A1Items(C.Structure):
    _fields_ = [("n_volume", _i64), ("n_interior", _i64), ("n_boundary", _i64), ("n_cols", _i64),
                ("volume_element", _p), ("face", _p), ("facet_row", _p), ("stripe_offset", _p),
                ("load_offset", _p)]


class AggOut(C.Structure):
    _fields_ = [(n, _p) for n in ("elem_ptr", "elem_simplices", "boxes", "elem_volumes", "face_owner",
                                  "face_neighbor", "face_normal", "face_measure", "face_ptr", "facet_vertices",
                                  "facet_owner_simplex", "facet_neighbor_simplex", "facet_measures",
                                  "iface_owner", "iface_neighbor", "iface_ptr", "elem_bface_ptr")] + \
               [("n_faces", _i64), ("n_facets", _i64), ("n_interfaces", _i64), ("n_interior_faces", _i64)]


class FaceItem(C.Structure):
    _fields_ = [("face", _i32), ("kind", _i32), ("upwind", _i32), ("pad_", _i32), ("sigma", C.c_double)]


UNIT_INTERIOR, UNIT_DIRICHLET, UNIT_INFLOW, UNIT_NEUMANN = 0, 1, 2, 3  # include/pdg.h PDG_UNIT_*

SLAB_MAX_DEGREE = {"P": 5, "PQ": 4}  # include/pdg.h PDG_SLAB_MAX_DEGREE(_PQ)

#: every symbol include/pdg.h declares (checked by the CPU test suite)
EXPORTS = ("pdg_abi_version", "pdg_last_error", "pdg_launch_count", "pdg_workspace_bytes", "pdg_adjacency",
           "pdg_pattern_offsets", "pdg_pattern_fill", "pdg_face_prepass", "pdg_iface_records", "pdg_frames_build",
           "pdg_assemble", "pdg_assemble_jit", "pdg_jit_prepare", "pdg_face_prepass_jit",
           "pdg_slab_prepare", "pdg_slab_prepass", "pdg_slab_assemble",
           "pdg_a1_emit", "pdg_triplets_workspace_bytes", "pdg_triplets_to_csr", "pdg_triplets_to_vector",
           "pdg_agglomerate_workspace_bytes", "pdg_agglomerate",
           "pdg_spmv_blocked", "pdg_block_jacobi_setup", "pdg_block_jacobi_apply",
           "pdg_map_simplices", "pdg_tabulate", "pdg_element_blocks", "pdg_face_blocks", "pdg_eval_coeffs",
           "pdg_host_alloc", "pdg_host_free", "pdg_pack_block_cols", "pdg_expand_block_cols")


class EngineUnavailable(RuntimeError):
    """The CUDA engine cannot run here (library or GPU missing)."""


@lru_cache(maxsize=1)
def load():
    """Load libpdg.so and declare prototypes."""
    if not os.path.exists(LIB_PATH):
        raise EngineUnavailable(
            f"{LIB_PATH} not built; run __graft_entry__.build() (no CPU fallback exists)")
    lib = C.CDLL(LIB_PATH)
    P = C.POINTER
    lib.pdg_abi_version.restype = C.c_int
    lib.pdg_last_error.restype = C.c_char_p
    lib.pdg_launch_count.restype = C.c_int64
    lib.pdg_workspace_bytes.restype = C.c_size_t
    lib.pdg_workspace_bytes.argtypes = [_i64, _i64]
    lib.pdg_adjacency.argtypes = [P(Mesh), _p, _p, _p, _p, C.c_size_t, _p]
    lib.pdg_pattern_offsets.argtypes = [P(Mesh), P(Basis), P(Pattern), _i64, P(_i64), _p,
                                        C.c_size_t, _p]
    lib.pdg_pattern_fill.argtypes = [P(Mesh), P(Basis), P(Pattern), _p]
    lib.pdg_face_prepass.argtypes = [P(Mesh), P(Basis), P(Coeffs), P(Rules), P(Params),
                                     _p, _p, _p, _p, _p]
    lib.pdg_iface_records.argtypes = [P(Mesh), P(Basis), P(Coeffs), P(Rules), P(Params), P(Pattern),
                                      _p, _p, _p]
    lib.pdg_frames_build.argtypes = [P(Mesh), P(Basis), P(Frames), _p, _p]
    lib.pdg_assemble.argtypes = [P(Mesh), P(Basis), P(Coeffs), P(Rules), P(Params), P(Pattern),
                                 P(Frames), _p, _p, _p, _i32, _p, _p, _p]
    lib.pdg_assemble_jit.argtypes = [P(Mesh), P(Basis), P(Coeffs), C.c_char_p, P(Rules), P(Params),
                                     P(Pattern), P(Frames), _p, _p, _p, _i32, _p, _p, _p]
    lib.pdg_face_prepass_jit.argtypes = [P(Mesh), P(Basis), P(Coeffs), C.c_char_p, P(Rules), P(Params),
                                         _p, _p, _p, _p, _p]
    lib.pdg_jit_prepare.argtypes = [P(Coeffs), C.c_char_p, _i32, _i32]
    lib.pdg_slab_prepare.argtypes = [C.c_char_p, _i32, _i32, _i32]
    lib.pdg_slab_prepass.argtypes = [P(Mesh), P(Basis), C.c_char_p, P(Rules), P(Params), P(Slab),
                                     P(Frames), _p, _p, _p, _p]
    lib.pdg_slab_assemble.argtypes = [P(Mesh), P(Basis), C.c_char_p, P(Rules), P(Params), P(Slab),
                                      P(Pattern), P(Frames), _p, _p, _p, _p, _p, _p]
    lib.pdg_a1_emit.argtypes = [P(Mesh), P(Basis), P(Coeffs), C.c_char_p, P(Rules), P(Params), P(Frames),
                                _p, _p, P(A1Items), _p, _p, _p, _p, _p, _p]
    lib.pdg_triplets_workspace_bytes.restype = C.c_size_t
    lib.pdg_triplets_workspace_bytes.argtypes = [_i64]
    lib.pdg_triplets_to_csr.argtypes = [_p, _p, _i64, _i64, _i64, _p, _p, _p, _p, _p, C.c_size_t, _p]
    lib.pdg_triplets_to_vector.argtypes = [_p, _p, _i64, _i64, _p, _p, C.c_size_t, _p]
    lib.pdg_agglomerate_workspace_bytes.restype = C.c_size_t
    lib.pdg_agglomerate_workspace_bytes.argtypes = [_i32, _i64, _i64]
    lib.pdg_agglomerate.argtypes = [_i32, _i64, _i64, _p, _p, _p, _p, _i64, _i32, P(AggOut), _p, C.c_size_t, _p]
    lib.pdg_spmv_blocked.argtypes = [_p, _i64, _p, _p, _p, _p, _p, _p, _p]
    lib.pdg_block_jacobi_setup.argtypes = [_p, _i64, _i32, _p, _p, _p, _p, _p, _p, _p]
    lib.pdg_block_jacobi_apply.argtypes = [_p, _i64, _p, _p, _p, _p, _p]
    lib.pdg_map_simplices.argtypes = [P(Mesh), P(Rules), _i32, _p, _i64, _p, _p, _p, _p]
    lib.pdg_tabulate.argtypes = [P(Mesh), P(Basis), _i32, _p, _i64, _p, _p, _p]
    lib.pdg_element_blocks.argtypes = [P(Mesh), P(Basis), P(Coeffs), P(Rules), P(Params),
                                       P(Frames), _p, _i64, _p, _p, _p, _p]
    lib.pdg_face_blocks.argtypes = [P(Mesh), P(Basis), P(Coeffs), P(Rules), P(Params), _p, _i64, _p, _p,
                                    _p, _p]
    lib.pdg_eval_coeffs.argtypes = [_i32, P(Coeffs), _p, _i64, _p, _p]
    lib.pdg_host_alloc.argtypes = [C.c_size_t, P(C.c_void_p)]
    lib.pdg_host_free.argtypes = [C.c_void_p]
    lib.pdg_pack_block_cols.argtypes = [_p, _p, _p, _p, _i64, _p, _p]
    lib.pdg_expand_block_cols.argtypes = [_i64, _p, _p, _p, _p, _i32]
    for name in EXPORTS:
        if name not in ("pdg_abi_version", "pdg_last_error", "pdg_launch_count", "pdg_workspace_bytes",
                        "pdg_triplets_workspace_bytes", "pdg_agglomerate_workspace_bytes"):
            getattr(lib, name).restype = C.c_int
    if lib.pdg_abi_version() != ABI_VERSION:
        raise EngineUnavailable("libpdg.so ABI version mismatch")
    return lib


def check(rc: int) -> None:
    """Map a C status code to the polydg-compatible exception classes."""
    if rc == PDG_OK:
        return
    msg = load().pdg_last_error().decode(errors="replace")
    if rc == PDG_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    if rc == PDG_ERR_CUDA:
        raise RuntimeError(f"CUDA error in libpdg: {msg}")
    raise ValueError(msg)


def ptr(t) -> int:
    """Device pointer of a torch tensor (0 for None)."""
    return 0 if t is None else int(t.data_ptr())


def stream_ptr(stream) -> int:
    return int(stream.cuda_stream) if stream is not None else 0


def coeffs_struct(desc) -> Coeffs:
    """Fill a ``pdg_coeffs`` from a compiled descriptor (model.compile_coeffs)."""
    c = Coeffs()
    c.diffusion_kind = desc["diffusion_kind"]
    c.diffusion_symmetric = desc["diffusion_symmetric"]
    c.has_advection = desc["has_advection"]
    c.has_reaction = desc["has_reaction"]
    c.has_source = desc["has_source"]
    c.has_dirichlet = desc["has_dirichlet"]
    c.has_neumann = desc["has_neumann"]

    def fill(dst, prog):
        dst.offset, dst.length, dst.is_const, dst.value = prog

    for i, pr in enumerate(desc["diffusion"]):
        fill(c.diffusion[i], pr)
    for i, pr in enumerate(desc["advection"]):
        fill(c.advection[i], pr)
    for name in ("reaction", "source", "dirichlet", "neumann"):
        if desc[name] is not None:
            fill(getattr(c, name), desc[name])
    code, consts = desc["code"], desc["consts"]
    c.n_code, c.n_const = len(code), len(consts)
    for i, v in enumerate(code):
        c.code[i] = v
    for i, v in enumerate(consts):
        c.consts[i] = v
    return c
