"""ctypes bindings of the product libraries (include/mswm_cuda.h, include/mswm_host.h).

The libraries are built in-tree by ``paper_2106_07154_b200/csrc/Makefile`` into
``paper_2106_07154_b200/_lib/``.  Nothing here falls back to Python: a missing
library raises immediately, so a GPU run can never silently take a CPU path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

LIB_DIR = Path(__file__).resolve().parent / "_lib"
HOST_LIB = LIB_DIR / "libmswm_host.so"
CUDA_LIB = Path(os.environ["MSWM_CUDA_LIB"]) if os.environ.get("MSWM_CUDA_LIB") else \
    LIB_DIR / "libmswm_cuda.so"

i32p = C.POINTER(C.c_int32)
i8p = C.POINTER(C.c_int8)
f64p = C.POINTER(C.c_double)
u8p = C.POINTER(C.c_uint8)
i64p = C.POINTER(C.c_int64)
u64p = C.POINTER(C.c_uint64)


class MeshDesc(C.Structure):
    """mswm_mesh_desc (include/mswm_cuda.h)."""

    _fields_ = [
        ("n_cells", C.c_int32),
        ("n_edges", C.c_int32),
        ("n_vertices", C.c_int32),
        ("cell_offset", i32p),
        ("cell_edges", i32p),
        ("cell_vertices", i32p),
        ("cell_cells", i32p),
        ("edge_cells", i32p),
        ("edge_vertices", i32p),
        ("vertex_cells", i32p),
        ("vertex_edges", i32p),
        ("edge_edge_offset", i32p),
        ("edge_edges", i32p),
        ("edge_cell_sign", i8p),
        ("edge_vertex_sign", i8p),
        ("edge_len", f64p),
        ("edge_dual_len", f64p),
        ("cell_area", f64p),
        ("vertex_area", f64p),
        ("vertex_kite", f64p),
        ("edge_weight", f64p),
    ]


class MeshSizes(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("n_cells", "n_edges", "n_vertices", "n_ring", "n_stencil")]


# (field, ctype pointer, numpy dtype, shape-kind) for every table of the desc.
DESC_TABLES = [
    ("cell_offset", i32p, np.int32, "C+1"),
    ("cell_edges", i32p, np.int32, "R"),
    ("cell_vertices", i32p, np.int32, "R"),
    ("cell_cells", i32p, np.int32, "R"),
    ("edge_cells", i32p, np.int32, "E2"),
    ("edge_vertices", i32p, np.int32, "E2"),
    ("vertex_cells", i32p, np.int32, "V3"),
    ("vertex_edges", i32p, np.int32, "V3"),
    ("edge_edge_offset", i32p, np.int32, "E+1"),
    ("edge_edges", i32p, np.int32, "S"),
    ("edge_cell_sign", i8p, np.int8, "E2"),
    ("edge_vertex_sign", i8p, np.int8, "E2"),
    ("edge_len", f64p, np.float64, "E"),
    ("edge_dual_len", f64p, np.float64, "E"),
    ("cell_area", f64p, np.float64, "C"),
    ("vertex_area", f64p, np.float64, "V"),
    ("vertex_kite", f64p, np.float64, "V3"),
    ("edge_weight", f64p, np.float64, "S"),
]


def table_shape(kind: str, nC: int, nE: int, nV: int, nR: int, nS: int):
    return {
        "C+1": (nC + 1,), "R": (nR,), "E2": (nE, 2), "V3": (nV, 3), "E+1": (nE + 1,),
        "S": (nS,), "E": (nE,), "C": (nC,), "V": (nV,),
    }[kind]


def as_ptr(arr: np.ndarray, ptype):
    assert arr.flags["C_CONTIGUOUS"], "tables must be C-contiguous"
    return arr.ctypes.data_as(ptype)


def view(ptr, dtype, shape):
    """Zero-copy numpy view of library memory (caller keeps the owner alive)."""
    n = int(np.prod(shape))
    if n == 0:
        return np.zeros(shape, dtype=dtype)
    addr = C.cast(ptr, C.c_void_p).value
    buf = (C.c_char * (n * np.dtype(dtype).itemsize)).from_address(addr)
    return np.frombuffer(buf, dtype=dtype).reshape(shape)


_host = None
_cuda = None


def _load(path: Path) -> C.CDLL:
    if not path.exists():
        raise RuntimeError(
            f"{path.name} is not built ({path}); run __graft_entry__.build() "
            "or `make -C paper_2106_07154_b200/csrc`")
    return C.CDLL(str(path), mode=C.RTLD_GLOBAL)


def host() -> C.CDLL:
    global _host
    if _host is None:
        lib = _load(HOST_LIB)
        lib.mswm_mesh_icosahedral.restype = C.c_void_p
        lib.mswm_mesh_icosahedral.argtypes = [C.c_int, C.c_double]
        lib.mswm_mesh_planar_hex.restype = C.c_void_p
        lib.mswm_mesh_planar_hex.argtypes = [C.c_int, C.c_int, C.c_double]
        lib.mswm_mesh_free.argtypes = [C.c_void_p]
        lib.mswm_mesh_free.restype = None
        lib.mswm_host_last_error.restype = C.c_char_p
        lib.mswm_mesh_get_sizes.argtypes = [C.c_void_p, C.POINTER(MeshSizes)]
        lib.mswm_mesh_get_desc.argtypes = [C.c_void_p, C.POINTER(MeshDesc)]
        lib.mswm_mesh_get_geometry.argtypes = [C.c_void_p] + [C.POINTER(f64p)] * 4
        lib.mswm_mesh_get_domain.argtypes = [C.c_void_p, C.POINTER(C.c_int), f64p, f64p, f64p]
        lib.mswm_mesh_locality_order.argtypes = [C.c_void_p, i32p]
        _host = lib
    return _host


def cuda() -> C.CDLL:
    """The CUDA drop-in library; raises if it is not built (no fallback)."""
    global _cuda
    if _cuda is None:
        lib = _load(CUDA_LIB)
        vp = C.c_void_p
        sig = {
            "mswm_cuda_create": (C.c_int, [C.POINTER(MeshDesc), C.c_int, i32p, C.POINTER(vp)]),
            "mswm_cuda_destroy": (None, [vp]),
            "mswm_cuda_last_error": (C.c_char_p, [vp]),
            "mswm_cuda_set_fields": (C.c_int, [vp, f64p, f64p, C.c_double]),
            "mswm_cuda_set_regions": (C.c_int, [vp, u8p, C.c_int, u8p, u8p, u8p, i64p,
                                                C.POINTER(C.c_int)]),
            "mswm_cuda_get_group": (C.c_int, [vp, C.c_int, i32p]),
            "mswm_cuda_get_closure": (C.c_int, [vp, C.c_uint, C.c_int, i32p, i64p]),
            "mswm_cuda_eval": (C.c_int, [vp, f64p, f64p, C.c_uint, f64p, f64p]),
            "mswm_cuda_state_upload": (C.c_int, [vp, f64p, f64p, C.c_double]),
            "mswm_cuda_state_download": (C.c_int, [vp, f64p, f64p, f64p]),
            "mswm_cuda_step": (C.c_int, [vp, C.c_int, C.c_double, C.c_int, C.c_int64, C.c_int]),
            "mswm_cuda_ledger": (C.c_int, [vp, i64p, i64p, i64p]),
            "mswm_cuda_ledger_reset": (C.c_int, [vp]),
            "mswm_cuda_dry_vertex": (C.c_int, [vp, i64p]),
            "mswm_cuda_sync": (C.c_int, [vp]),
            "mswm_cuda_stream": (vp, [vp]),
            "mswm_cuda_set_profiling": (C.c_int, [vp, C.c_int]),
            "mswm_cuda_eval_profile": (C.c_int, [vp, C.POINTER(C.c_float), i64p, i64p, C.c_int,
                                                 C.POINTER(C.c_int)]),
            "mswm_cuda_total_mass": (C.c_int, [vp, f64p]),
            "mswm_cuda_diagnostics": (C.c_int, [vp, C.c_int, f64p, f64p]),
            "mswm_cuda_courant": (C.c_int, [vp, C.c_double, C.c_int, f64p, f64p]),
            "mswm_cuda_halo_needs": (C.c_int, [vp, C.c_uint, i64p, i32p]),
            "mswm_cuda_set_halo_mask": (C.c_int, [vp, C.c_uint, i64p, i32p, i64p, i32p]),
            "mswm_cuda_kernels_per_step": (C.c_int, [vp, i64p]),
            "mswm_cuda_schedule_info": (C.c_int, [vp, C.POINTER(C.c_int)]),
            "mswm_cuda_set_replication": (C.c_int, [vp, C.c_int]),
            "mswm_cuda_layout_info": (C.c_int, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
            "mswm_cuda_stencil_info": (C.c_int, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int64)]),
            "mswm_cuda_index_info": (C.c_int, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int64),
                                               C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
            "mswm_cuda_set_labels": (C.c_int, [vp, u8p, u8p, u8p, u8p, u8p, C.c_int]),
            "mswm_cuda_validate_labels": (C.c_int, [vp, u8p, u8p, u8p, C.c_int, i64p, i32p]),
            "mswm_cuda_set_halo": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, i32p, i64p, i32p]),
            "mswm_cuda_nccl_unique_id": (C.c_int, [vp]),
            "mswm_cuda_comm_init": (C.c_int, [vp, vp, C.c_int, C.c_int]),
            "mswm_cuda_group_create": (C.c_int, [C.POINTER(vp), C.c_int, C.POINTER(vp)]),
            "mswm_cuda_group_destroy": (None, [vp]),
            "mswm_cuda_group_step": (C.c_int, [vp, C.c_int, C.c_double, C.c_int, C.c_int64]),
            "mswm_cuda_halo_reach": (C.c_int, [vp, i32p, C.c_int, u64p, u64p, u64p]),
            "mswm_cuda_partition": (C.c_int, [vp, i32p, C.c_int, i32p, i32p]),
            "mswm_cuda_group_nccl_loopback": (C.c_int, [vp]),
            "mswm_cuda_group_peer": (C.c_int, [vp, C.c_int]),
            "mswm_cuda_peer_export": (C.c_int, [vp, vp, i64p, C.c_int64, i64p]),
            "mswm_cuda_peer_import": (C.c_int, [vp, C.c_int, vp, i64p, C.c_int64]),
            "mswm_cuda_peer_enable": (C.c_int, [vp, C.c_int]),
            "mswm_cuda_peer_exchange": (C.c_int, [vp, C.c_int]),
            "mswm_cuda_group_last_error": (C.c_char_p, [vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _cuda = lib
    return _cuda


def header_symbols(header: Path) -> list[str]:
    """Function names declared in one of include/*.h (for the export test)."""
    import re

    text = header.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mswm_[a-z0-9_]+)\s*\(", text)))


REPO_ROOT = Path(__file__).resolve().parent.parent
INCLUDE_DIR = REPO_ROOT / "include"

os.environ.setdefault("CUDA_MODULE_LOADING", "LAZY")
