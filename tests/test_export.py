"""export.hpp formats (voxel listing, OBJ mesh) and the CLI front end's
argument handling (voxevo_main.cpp) — host-only.  The cases restate the
reference's own tests (test_export.cpp:33-114)."""
import numpy as np
import pytest

from paper_2405_00698_b200.export import ExportError, export_voxel_listing, mesh_obj, voxel_listing


def _two_voxel():
    # VoxelGrid(2,1,1): (0,0,0) MuscleExpand 0.75, (1,0,0) HardBone 1.0
    return np.array([1, 4], np.uint8), np.array([0.75, 1.0]), 2, 1, 1


def test_voxel_listing_prints_occupied_cells_with_material_ids():
    lines = voxel_listing(*_two_voxel()).splitlines()
    assert lines == ["# x y z material weight", "0 0 0 1 0.75", "1 0 0 4 1"]


def test_voxel_listing_skips_empty_cells():
    m = np.zeros(27, np.uint8)
    w = np.zeros(27)
    i = 2 + 3 * (1 + 3 * 0)
    m[i], w[i] = 3, 0.5
    lines = voxel_listing(m, w, 3, 3, 3).splitlines()
    assert len(lines) == 2 and lines[1] == "2 1 0 3 0.5"


def test_voxel_listing_full_precision_weights():
    m = np.array([2], np.uint8)
    assert voxel_listing(m, np.array([0.123456789123]), 1, 1, 1).splitlines()[1] == "0 0 0 2 0.123456789"


def test_obj_one_cube_per_voxel_grouped_by_material():
    m, _, w, h, d = _two_voxel()
    obj = mesh_obj(m, w, h, d, 0.1)
    lines = obj.splitlines()
    v = [ln for ln in lines if ln.startswith("v ")]
    f = [ln for ln in lines if ln.startswith("f ")]
    g = [ln for ln in lines if ln.startswith("g ")]
    assert len(v) == 16 and len(f) == 12 and len(g) == 2
    idx = [int(t) for ln in f for t in ln.split()[1:]]
    assert all(len(ln.split()) == 5 for ln in f) and min(idx) >= 1 and max(idx) == len(v)
    assert "g muscle_expand" in obj and "g hard_bone" in obj and "usemtl muscle_expand" in obj
    assert lines[0] == "# voxevo robot mesh, cube edge 0.100000 m"
    # groups follow the material order, not the scan order
    assert obj.index("g muscle_expand") < obj.index("g hard_bone")


def test_obj_faces_wind_outward():
    obj = mesh_obj(np.array([3], np.uint8), 1, 1, 1, 1.0)
    verts = [tuple(map(float, ln.split()[1:])) for ln in obj.splitlines() if ln.startswith("v ")]
    faces = [tuple(map(int, ln.split()[1:])) for ln in obj.splitlines() if ln.startswith("f ")]
    assert len(verts) == 8 and len(faces) == 6
    for fa in faces:
        a, b, c = (np.array(verts[i - 1]) for i in fa[:3])
        n = np.cross(b - a, c - a)
        assert np.dot(n, a - 0.5) > 0


def test_export_error_on_unwritable_path(tmp_path):
    with pytest.raises(ExportError, match="cannot open for writing"):
        export_voxel_listing(str(tmp_path / "missing" / "v.txt"), *_two_voxel())


def test_cli_rejects_bad_arguments(capsys):
    from paper_2405_00698_b200.runner import main
    with pytest.raises(SystemExit):
        main(["bench", "--jobs", "0"])
    with pytest.raises(SystemExit):
        main(["run", "--advisor", "sometimes"])
    with pytest.raises(SystemExit):
        main(["export-mesh", "--genome", "/nonexistent/g.json"])
    with pytest.raises(SystemExit):
        main(["resume"])  # --checkpoint is required
