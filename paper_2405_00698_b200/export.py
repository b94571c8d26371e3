"""export-mesh / voxel listing (export.hpp:17-86) for device-decoded grids.

A grid here is the decode layout: ``materials`` (cells u8) and ``weights``
(cells f64) with cell index x + w(y + h z) (morphology.hpp:83).  Formats are
the reference's byte for byte: the listing prints ``x y z material weight``
with ``%.9g`` weights; the OBJ writes one 8-vertex cube per occupied voxel,
``%.6f`` coordinates, one ``g``/``usemtl`` group per solid material in the
order muscle_expand, muscle_contract, soft_tissue, hard_bone, faces wound
counter-clockwise seen from outside.
"""
from __future__ import annotations

import numpy as np

MATERIAL_NAMES = ("empty", "muscle_expand", "muscle_contract", "soft_tissue", "hard_bone")  # morphology.hpp:33-42
_FACES = ((0, 3, 2, 1), (4, 5, 6, 7), (0, 1, 5, 4), (2, 3, 7, 6), (0, 4, 7, 3), (1, 2, 6, 5))


class ExportError(RuntimeError):
    """export_error (export.hpp:14-16)."""


def _cells(materials, w, h, d):
    m = np.asarray(materials, np.uint8).reshape(-1)
    if m.size != w * h * d:
        raise ValueError("grid size does not match w*h*d")
    return m


def voxel_listing(materials, weights, w: int, h: int, d: int) -> str:
    """write_voxel_listing (export.hpp:28-41)."""
    m = _cells(materials, w, h, d)
    wt = np.asarray(weights, np.float64).reshape(-1)
    out = ["# x y z material weight\n"]
    for z in range(d):
        for y in range(h):
            for x in range(w):
                i = x + w * (y + h * z)
                if m[i] == 0:
                    continue
                out.append("%d %d %d %d %s\n" % (x, y, z, m[i], "%.9g" % wt[i]))
    return "".join(out)


def mesh_obj(materials, w: int, h: int, d: int, voxel_edge: float) -> str:
    """write_mesh_obj (export.hpp:46-86)."""
    m = _cells(materials, w, h, d)
    out = ["# voxevo robot mesh, cube edge %.6f m\n" % voxel_edge]
    nv = 1
    for mat in (1, 2, 3, 4):
        group_open = False
        for z in range(d):
            for y in range(h):
                for x in range(w):
                    if m[x + w * (y + h * z)] != mat:
                        continue
                    if not group_open:
                        out.append("g %s\nusemtl %s\n" % (MATERIAL_NAMES[mat], MATERIAL_NAMES[mat]))
                        group_open = True
                    x0, x1 = x * voxel_edge, (x + 1) * voxel_edge
                    y0, y1 = y * voxel_edge, (y + 1) * voxel_edge
                    z0, z1 = z * voxel_edge, (z + 1) * voxel_edge
                    for c in ((x0, y0, z0), (x1, y0, z0), (x1, y1, z0), (x0, y1, z0),
                              (x0, y0, z1), (x1, y0, z1), (x1, y1, z1), (x0, y1, z1)):
                        out.append("v %.6f %.6f %.6f\n" % c)
                    for f in _FACES:
                        out.append("f %d %d %d %d\n" % (nv + f[0], nv + f[1], nv + f[2], nv + f[3]))
                    nv += 8
    return "".join(out)


def _write(path: str, text: str):
    try:
        with open(path, "wb") as f:
            f.write(text.encode())
    except OSError as e:
        raise ExportError(("cannot open for writing: " if isinstance(e, (FileNotFoundError, PermissionError,
                                                                        IsADirectoryError))
                           else "write failed: ") + path) from e


def export_voxel_listing(path: str, materials, weights, w: int, h: int, d: int):
    """export_voxel_listing (export.hpp:72-77)."""
    _write(path, voxel_listing(materials, weights, w, h, d))


def export_mesh_obj(path: str, materials, w: int, h: int, d: int, voxel_edge: float):
    """export_mesh_obj (export.hpp:79-84)."""
    _write(path, mesh_obj(materials, w, h, d, voxel_edge))
