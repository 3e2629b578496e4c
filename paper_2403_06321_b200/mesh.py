"""Tet meshes, incidence and the device colouring front-end.

Mirrors pkg/src/vbdsim/mesh.py (TetMesh, build_tet_mesh, incidence,
VertexAdjacency, ColorPartition, greedy_color) and the procedural generators of
pkg/src/vbdsim/harness.py:28-76.  The host side is NumPy (one-off set-up);
``greedy_color`` runs the K5 Jones-Plassmann kernel on the GPU and returns the
reference's greedy colouring bit-exactly.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import DegenerateTet, IndexOutOfRange

_TET_FACES = ((0, 2, 1), (0, 1, 3), (1, 2, 3), (0, 3, 2))

# 5-tet split of a hex cell alternated by parity; corner index 4 dx + 2 dy + dz
# (harness.py:30-33)
_CELL_EVEN = np.array(((0, 3, 5, 6), (1, 0, 3, 5), (2, 0, 3, 6), (4, 0, 5, 6), (7, 3, 5, 6)))
_CELL_ODD = np.array(((1, 2, 4, 7), (0, 1, 2, 4), (3, 1, 2, 7), (5, 1, 4, 7), (6, 2, 4, 7)))


@dataclass(frozen=True)
class TetMesh:
    rest_positions: np.ndarray
    tets: np.ndarray
    surface_tris: np.ndarray
    surface_edges: np.ndarray
    rest_volumes: np.ndarray
    inv_rest_shape: np.ndarray
    masses: np.ndarray
    density: float

    @property
    def num_vertices(self) -> int:
        return len(self.rest_positions)

    @property
    def num_tets(self) -> int:
        return len(self.tets)

    def bbox_diagonal(self) -> float:
        return float(np.linalg.norm(self.rest_positions.max(0) - self.rest_positions.min(0)))


@dataclass(frozen=True)
class SpringNet:
    """Particles joined by linear springs (mesh.py:60-79): row s is (indices[s],
    rest_length[s], stiffness[s])."""

    particles: np.ndarray
    indices: np.ndarray
    rest_length: np.ndarray
    stiffness: np.ndarray
    masses: np.ndarray

    @property
    def num_vertices(self) -> int:
        return len(self.particles)

    @property
    def num_springs(self) -> int:
        return len(self.indices)


@dataclass(frozen=True)
class VertexAdjacency:
    num_vertices: int
    elem_offsets: np.ndarray
    elem_ids: np.ndarray
    elem_slots: np.ndarray
    neighbor_offsets: np.ndarray
    neighbor_ids: np.ndarray

    def elements_of(self, i):
        return self.elem_ids[self.elem_offsets[i]:self.elem_offsets[i + 1]]

    def neighbors_of(self, i):
        return self.neighbor_ids[self.neighbor_offsets[i]:self.neighbor_offsets[i + 1]]

    def degree(self, i) -> int:
        return int(self.neighbor_offsets[i + 1] - self.neighbor_offsets[i])


@dataclass(frozen=True)
class ColorPartition:
    color_of: np.ndarray
    groups: tuple
    num_colors: int

    def group(self, c):
        return self.groups[c]


def build_tet_mesh(rest_positions, tets, density: float) -> TetMesh:
    """mesh.py:128-170: orientation fix, |V|, Dm^-1, lumped masses rho V / 4."""
    pos = np.ascontiguousarray(rest_positions, dtype=np.float64)
    tets = np.ascontiguousarray(tets, dtype=np.int64)
    if pos.ndim != 2 or pos.shape[1] != 3 or len(pos) < 4:
        raise ValueError("rest_positions must be (N,3) with N >= 4")
    if tets.ndim != 2 or tets.shape[1] != 4:
        raise ValueError("tets must be (T,4)")
    if density <= 0.0:
        raise ValueError("density must be positive")
    n = len(pos)
    if tets.size and (tets.min() < 0 or tets.max() >= n):
        raise IndexOutOfRange(f"tet index outside [0,{n})")
    d = pos[tets[:, 1:]] - pos[tets[:, :1]]
    vol = np.linalg.det(np.swapaxes(d, 1, 2)) / 6.0
    flip = vol < 0.0
    if np.any(flip):
        tets = tets.copy()
        tets[flip] = tets[flip][:, [0, 2, 1, 3]]
        vol = np.abs(vol)
    diag = float(np.linalg.norm(pos.max(axis=0) - pos.min(axis=0)))
    if np.any(vol <= 1e-12 * diag ** 3):
        bad = int(np.argmin(vol))
        raise DegenerateTet(f"tet {bad} has volume {vol[bad]:.3e}")
    d_m = np.swapaxes(pos[tets[:, 1:]] - pos[tets[:, :1]], 1, 2)
    inv = np.linalg.inv(d_m)
    masses = np.zeros(n)
    np.add.at(masses, tets.ravel(), np.repeat(density * vol / 4.0, 4))
    faces = np.concatenate([tets[:, f] for f in _TET_FACES])
    key = np.sort(faces, axis=1)
    _, first, counts = np.unique(key, axis=0, return_index=True, return_counts=True)
    boundary = faces[first[counts == 1]]
    surf = np.ascontiguousarray(boundary[np.lexsort((boundary[:, 2], boundary[:, 1], boundary[:, 0]))])
    if len(surf):
        e = np.concatenate([surf[:, [0, 1]], surf[:, [1, 2]], surf[:, [2, 0]]])
        edges = np.ascontiguousarray(np.unique(np.sort(e, axis=1), axis=0))
    else:
        edges = np.zeros((0, 2), dtype=np.int64)
    for a in (pos, tets, surf, edges, vol, inv, masses):
        a.setflags(write=False)
    return TetMesh(pos, tets, surf, edges, vol, inv, masses, float(density))


def beam_connectivity(nx: int, ny: int, nz: int) -> np.ndarray:
    """generate_beam's tets (harness.py:54-66) without the Python triple loop."""
    cx, cy, cz = np.meshgrid(np.arange(nx - 1), np.arange(ny - 1), np.arange(nz - 1), indexing="ij")
    cx, cy, cz = cx.ravel(), cy.ravel(), cz.ravel()
    corner = np.empty((len(cx), 8), dtype=np.int64)
    for dx in (0, 1):
        for dy in (0, 1):
            for dz in (0, 1):
                corner[:, dx * 4 + dy * 2 + dz] = ((cx + dx) * ny + (cy + dy)) * nz + (cz + dz)
    even = ((cx + cy + cz) % 2 == 0)[:, None, None]
    pat = np.where(even, _CELL_EVEN[None], _CELL_ODD[None])  # (cells, 5, 4)
    tets = np.take_along_axis(corner[:, None, :].repeat(5, axis=1), pat, axis=2)
    return np.ascontiguousarray(tets.reshape(-1, 4))


def generate_beam(nx: int, ny: int, nz: int, spacing: float, density: float = 1000.0) -> TetMesh:
    """harness.py:42-67."""
    if min(nx, ny, nz) < 2:
        raise ValueError("beam needs at least 2 vertices per axis")
    if spacing <= 0.0:
        raise ValueError("spacing must be positive")
    ix, iy, iz = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    pos = spacing * np.stack([ix, iy, iz], axis=-1).reshape(-1, 3).astype(np.float64)
    return build_tet_mesh(pos, beam_connectivity(nx, ny, nz), density)


def generate_cube(n: int, edge: float, density: float = 1000.0) -> TetMesh:
    """harness.py:70-76."""
    if n < 2:
        raise ValueError("cube needs n >= 2")
    if edge <= 0.0:
        raise ValueError("edge must be positive")
    return generate_beam(n, n, n, edge / (n - 1), density)


def build_spring_net(particles, springs, masses) -> SpringNet:
    """mesh.py:192-215: springs rows are (i, j, rest_length, stiffness)."""
    particles = np.ascontiguousarray(particles, dtype=np.float64)
    masses = np.ascontiguousarray(masses, dtype=np.float64)
    springs = np.asarray(springs, dtype=np.float64).reshape(-1, 4)
    idx = np.ascontiguousarray(springs[:, :2].astype(np.int64))
    l0 = np.ascontiguousarray(springs[:, 2])
    k = np.ascontiguousarray(springs[:, 3])
    n = len(particles)
    if idx.size and (idx.min() < 0 or idx.max() >= n):
        raise IndexOutOfRange(f"spring index outside [0,{n})")
    if np.any(idx[:, 0] == idx[:, 1]):
        raise ValueError("spring endpoints must be distinct")
    if np.any(l0 <= 0.0):
        raise ValueError("rest lengths must be positive")
    if np.any(k < 0.0):
        raise ValueError("stiffness must be >= 0")
    if np.any(masses <= 0.0):
        raise ValueError("masses must be positive")
    return SpringNet(particles, idx, l0, k, masses)


def generate_chain(count: int, spacing: float, stiffness: float, mass: float = 1.0) -> SpringNet:
    """harness.py:79-90: `count` particles hanging along -y, linked by serial springs."""
    if count < 2:
        raise ValueError("chain needs at least 2 particles")
    if spacing <= 0.0 or stiffness <= 0.0 or mass <= 0.0:
        raise ValueError("spacing, stiffness and mass must be positive")
    particles = np.zeros((count, 3))
    particles[:, 1] = -spacing * np.arange(count)
    springs = [[i, i + 1, spacing, stiffness] for i in range(count - 1)]
    return build_spring_net(particles, springs, np.full(count, mass))


def load_node_ele(node_path, ele_path) -> tuple:
    """mesh.py:305-333: ``.node`` rows ``index x y z`` (indices 0..N-1 in order) and ``.ele``
    rows ``index v0 v1 v2 v3``, 0-based; blank and ``#`` lines skipped; extra columns
    ignored.  Returns (positions (N,3) float64, tets (T,4) int64) for build_tet_mesh."""

    def table(path, cols):
        rows = []
        with open(path, encoding="utf-8") as fh:
            for no, raw in enumerate(fh, 1):
                line = raw.strip()
                if line and not line.startswith("#"):
                    fields = line.split()
                    if len(fields) < cols:
                        raise ValueError(f"{path}:{no}: expected {cols} columns")
                    rows.append(fields[:cols])
        return np.array(rows, dtype=np.float64).reshape(-1, cols)

    nodes = table(node_path, 4)
    if not np.array_equal(nodes[:, 0].astype(np.int64), np.arange(len(nodes))):
        raise ValueError(f"{node_path}: node indices must be 0..N-1 in order")
    eles = table(ele_path, 5)
    return np.ascontiguousarray(nodes[:, 1:]), np.ascontiguousarray(eles[:, 1:].astype(np.int64))


def incidence_from_elements(elements, num_vertices: int) -> VertexAdjacency:
    """mesh.py:232-267."""
    elements = np.asarray(elements, dtype=np.int64)
    n = num_vertices
    if elements.size == 0:
        z = np.zeros(n + 1, dtype=np.int64)
        e = np.zeros(0, dtype=np.int64)
        return VertexAdjacency(n, z, e, e.copy(), z.copy(), e.copy())
    num, arity = elements.shape
    verts = elements.ravel()
    eids = np.repeat(np.arange(num, dtype=np.int64), arity)
    slots = np.tile(np.arange(arity, dtype=np.int64), num)
    order = np.lexsort((eids, verts))
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(verts, minlength=n), out=off[1:])
    noff, nids = merged_adjacency(n, [elements])
    return VertexAdjacency(n, off, np.ascontiguousarray(eids[order]),
                           np.ascontiguousarray(slots[order]), noff, nids)


def incidence(mesh) -> VertexAdjacency:
    if isinstance(mesh, TetMesh):
        return incidence_from_elements(mesh.tets, mesh.num_vertices)
    if isinstance(mesh, SpringNet):
        return incidence_from_elements(mesh.indices, mesh.num_vertices)
    raise TypeError(f"unsupported mesh type {type(mesh)!r}")


def merged_adjacency(n: int, element_arrays):
    """Distinct-neighbour CSR over all element vertex pairs (_system.py:147-169)."""
    pairs = []
    for el in element_arrays:
        el = np.asarray(el, dtype=np.int64)
        if len(el) == 0:
            continue
        pa, pb = np.triu_indices(el.shape[1], k=1)
        u, v = el[:, pa].ravel(), el[:, pb].ravel()
        pairs.append(np.stack([np.concatenate([u, v]), np.concatenate([v, u])], axis=1))
    uniq = np.unique(np.concatenate(pairs), axis=0) if pairs else np.zeros((0, 2), np.int64)
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(uniq[:, 0], minlength=n), out=off[1:])
    return off, np.ascontiguousarray(uniq[:, 1])


def greedy_color(adjacency: VertexAdjacency, order=None, device: int = 0) -> ColorPartition:
    """greedy_color (mesh.py:270-302) computed on the GPU by K5 (vbd_greedy_color).

    Jones-Plassmann with the greedy visiting order as the priority: bit-identical
    to the reference's sequential greedy for any graph and order.
    """
    n = adjacency.num_vertices
    noff = _lib.i64c(adjacency.neighbor_offsets)
    nids = _lib.i64c(adjacency.neighbor_ids)
    o = None
    if order is not None:
        o = _lib.i64c(order)
        if o.shape != (n,) or not np.array_equal(np.sort(o), np.arange(n)):
            raise ValueError("order must be a permutation of all vertices")
    col = np.empty(n, dtype=np.int64)
    nc = ctypes.c_int64(0)
    _lib.check(_lib.lib().vbd_greedy_color(n, _lib.ptr(noff), _lib.ptr(nids), _lib.ptr(o), device,
                                           _lib.ptr(col), ctypes.byref(nc)))
    groups = tuple(np.flatnonzero(col == c) for c in range(nc.value))
    col.setflags(write=False)
    for g in groups:
        g.setflags(write=False)
    return ColorPartition(col, groups, nc.value)
