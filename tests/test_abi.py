"""The C-ABI libraries load and export every symbol their headers declare
(no compute calls: this runs on CPU-only hosts too)."""
import ctypes

from paper_2106_07154_b200 import _lib


def _exports(lib_path, header):
    lib = ctypes.CDLL(str(lib_path))
    missing = [s for s in _lib.header_symbols(header) if not hasattr(lib, s)]
    return missing


def test_cuda_library_exports_header():
    names = _lib.header_symbols(_lib.INCLUDE_DIR / "mswm_cuda.h")
    assert "mswm_cuda_eval" in names and "mswm_cuda_step" in names and len(names) >= 18
    assert _exports(_lib.CUDA_LIB, _lib.INCLUDE_DIR / "mswm_cuda.h") == []


def test_host_library_exports_header():
    assert _exports(_lib.HOST_LIB, _lib.INCLUDE_DIR / "mswm_host.h") == []


def test_python_bindings_cover_the_header():
    lib = _lib.cuda()
    for s in _lib.header_symbols(_lib.INCLUDE_DIR / "mswm_cuda.h"):
        assert getattr(lib, s).argtypes is not None, s


def test_cuda_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.CUDA_LIB)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_create_without_gpu_fails_cleanly():
    import torch
    if torch.cuda.is_available():
        return
    from paper_2106_07154_b200.api import CudaContext, Error
    from paper_2106_07154_b200.mesh import Mesh
    import numpy as np
    import pytest
    m = Mesh.icosahedral(1, 1.0)
    with pytest.raises(Error):
        CudaContext(m, np.zeros(m.n_cells), np.zeros(m.n_vertices))
