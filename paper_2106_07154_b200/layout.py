"""Device-layout helpers (host side).

``region_major_order`` builds a cell order for ``mswm_cuda_create`` that
groups cells by LTS region class -- plain fine, UF1, UF2, Interface1,
Interface2, coarse, i.e. GroupBit order -- and keeps the space-filling-curve
order inside each class.  Every group list then becomes one contiguous range
of internal ids, and so does every LTS mask's output set (edges and vertices
are sorted by their lowest cell, so their groups follow).  The labels are a
numpy restatement of make_regions (regions.cpp:69-139) used only as a layout
hint: results never depend on the layout (the library re-derives the labels
bit-exactly on the device).
"""
from __future__ import annotations

import numpy as np

from .mesh import Mesh


def region_keys(mesh: Mesh, fine_mask: np.ndarray, width: int = 1) -> np.ndarray:
    """GroupBit cell index (0 plain fine .. 5 coarse) per cell."""
    n = mesh.n_cells
    deg = np.diff(mesh.cell_offset)
    rows = np.repeat(np.arange(n), deg)
    nbr = mesh.cell_cells
    dist = np.where(np.asarray(fine_mask) != 0, 0, -1).astype(np.int64)
    for level in range(1, 2 * width + 1):
        hit = np.zeros(n, bool)
        hit[rows[dist[nbr] == level - 1]] = True
        dist[(dist == -1) & hit] = level
    key = np.full(n, 5, np.int8)
    key[(dist >= 1) & (dist <= width)] = 3
    key[(dist > width) & (dist <= 2 * width)] = 4
    fine = dist == 0
    key[fine] = 0
    # underline layers: fine cells touching Interface1, then fine cells
    # touching those (regions.cpp:107-139)
    touch = np.zeros(n, bool)
    touch[rows[key[nbr] == 3]] = True
    uf1 = fine & touch
    key[uf1] = 1
    touch[:] = False
    touch[rows[uf1[nbr]]] = True
    key[fine & ~uf1 & touch] = 2
    return key


def region_major_order(mesh: Mesh, fine_mask: np.ndarray, width: int = 1,
                       base_order: np.ndarray | None = None) -> np.ndarray:
    """Cells grouped by region class, ``base_order`` (default: the Hilbert
    locality order) inside each class."""
    base = mesh.locality_order() if base_order is None else np.asarray(base_order)
    key = region_keys(mesh, fine_mask, width)
    return base[np.argsort(key[base], kind="stable")].astype(np.int32)
