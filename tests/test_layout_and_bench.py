"""CPU tests of the host-side helpers: region-major layout hint (a numpy
restatement of make_regions) and the bench contract's reference arm."""
import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle.oracle import Oracle
from paper_2106_07154_b200 import workloads as W
from paper_2106_07154_b200.layout import region_keys, region_major_order

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("make", [lambda: W.config1(n_steps=1),
                                  lambda: W.small_sphere(5, cap_deg=25.0)])
@pytest.mark.parametrize("width", [1, 2])
def test_region_keys_match_oracle_labels(make, width):
    wl = make()
    o = Oracle(wl.mesh, wl.b, wl.f, wl.gravity)
    o.set_regions(wl.fine_mask, width)
    cl, cs, el = o.labels()
    ref = np.where(cl == 0, cs, cl + 2)
    assert np.array_equal(region_keys(wl.mesh, wl.fine_mask, width), ref)


def test_region_major_order_is_grouped_permutation():
    wl = W.small_sphere(4, cap_deg=30.0)
    order = region_major_order(wl.mesh, wl.fine_mask)
    assert np.array_equal(np.sort(order), np.arange(wl.mesh.n_cells))
    keys = region_keys(wl.mesh, wl.fine_mask)[order]
    assert np.all(np.diff(keys) >= 0)  # groups are contiguous, in GroupBit order


def test_bench_reference_arm_json_line():
    """`bench.py --impl reference` prints one JSON line with the contract keys."""
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config",
                        "c1", "--steps", "2", "--warmup", "3"], capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference"
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def test_bench_reference_arm_maps_no_product_library():
    """The spherical reference arm builds its mesh with the reference's own
    generator and runs the reference's Stepper: only oracle/ libraries are
    mapped (no libmswm_cuda / libmswm_host), and it runs the requested step
    count plus the 1-core SerialEvaluator leg."""
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config",
                        "c4", "--level", "4", "--steps", "3", "--warmup", "3"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][0])
    libs = d["repo_libraries_loaded"]
    assert libs and all(p.startswith("oracle/") for p in libs), libs
    assert not any("dropin" in p for p in libs), libs
    assert d["steps"] == 3 and d["warmup"] == 3
    assert d["cpu_baseline"]["serial_1core"]["cores"] == 1
    assert d["cpu_baseline"]["host"]["nproc"] >= 1
    assert "reference build_voronoi_mesh" in d["cpu_baseline"]["sample"]


@pytest.mark.slow
def test_reference_builder_equals_ours_at_level10():
    """The reference arm's C4 mesh (the reference's build_voronoi_mesh at
    level 10) is bitwise the mesh our builder gives the GPU path."""
    from oracle.oracle import RefMesh, ref_available
    from paper_2106_07154_b200.mesh import Mesh
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    ours = Mesh.icosahedral(10, W.EARTH_RADIUS).digest()
    theirs = RefMesh.icosahedral(10, W.EARTH_RADIUS).as_mesh().digest()
    assert ours == theirs


def test_bench_ours_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--config", "c1", "--steps", "2"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode != 0 and "CUDA" in (r.stderr + r.stdout)


def test_bench_reference_ranks_fit_host_memory(monkeypatch):
    """The CPU baseline sizes the reference's ThreadedEvaluator to host RAM
    (3 full-size blocks per rank, rank_pool.cpp:93-95): all threads when they
    fit, fewer ranks, SerialEvaluator, or 'unavailable' -- never an OOM kill."""
    from types import SimpleNamespace as NS
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import bench
    c4 = NS(mesh=NS(n_cells=10485762, n_edges=31457280))
    c5 = NS(mesh=NS(n_cells=41943042, n_edges=125829120))
    monkeypatch.setattr(bench, "_mem_available", lambda: 196e9)
    assert bench.ref_ranks(c4, 16) == (16, "")
    r, note = bench.ref_ranks(c5, 16)
    assert 2 <= r < 16 and "host RAM" in note
    assert 3 * r * 36.0 * (c5.mesh.n_cells + c5.mesh.n_edges) <= 0.5 * 196e9
    monkeypatch.setattr(bench, "_mem_available", lambda: 62e9)
    assert bench.ref_ranks(c5, 16)[0] == 0
    monkeypatch.setattr(bench, "_mem_available", lambda: 8e9)
    assert bench.ref_ranks(c5, 16)[0] is None
