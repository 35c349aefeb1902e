"""Quad meshes: the host-side input provider for the device residual.

Mirrors the data format of the reference's ``pmgflow.mesh``
(``/root/reference/pkg/src/pmgflow/mesh.py``) so that a mesh built by
either package means the same thing to the kernels:

* ``Mesh`` fields (mesh.py:31-63): ``nodes`` (Nn,2), ``elements`` (M,4)
  CCW corners, ``interior_faces`` (Nf,5) rows (eL, fL, eR, fR, rev),
  sorted; ``boundary_faces`` (Nb,2) rows (e, f) sorted, with a tag each.
* local face f joins corners FACE_NODES[f] = (0,1),(1,2),(2,3),(3,0)
  (mesh.py:22); a shared face is "reversed" when the two CCW
  traversals run opposite ways (mesh.py:104-110); periodic pairs are
  appended as reversed interior faces (mesh.py:112-116).
* ``generate_box`` (mesh.py:139-172) and ``generate_cylinder_omesh``
  (mesh.py:175-221) numbering.
* ``element_geometry`` (mesh.py:322-395): bilinear metrics at the
  Gauss points, unit outward normals and face_jac = |edge|/2.

Mesh generation is one-time host setup; the device only ever sees the
packed arrays built by ``pack_geometry`` / ``pack_links``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .operators import basis

FACE_NODES = ((0, 1), (1, 2), (2, 3), (3, 0))
BOUNDARY_TAGS = ("wall-adiabatic", "wall-slip", "far-field", "wall-isothermal")
TAG_CODE = {t: i for i, t in enumerate(BOUNDARY_TAGS)}


class MeshError(Exception):
    """Invalid mesh topology or geometry."""


@dataclass(frozen=True)
class Mesh:
    nodes: np.ndarray
    elements: np.ndarray
    interior_faces: np.ndarray
    boundary_faces: np.ndarray
    boundary_tags: tuple

    @property
    def n_elements(self) -> int:
        return int(self.elements.shape[0])

    def element_corners(self, e: int) -> np.ndarray:
        return self.nodes[self.elements[e]]

    def edge_lengths(self) -> np.ndarray:
        xy = self.nodes[self.elements]
        d = np.roll(xy, -1, axis=1) - xy
        return np.hypot(d[..., 0], d[..., 1])

    @property
    def h_min(self) -> float:
        return float(self.edge_lengths().min())


def _shape_derivs(xi, eta):
    """dN/dxi, dN/deta of the Q1 shape functions, corners CCW from (-1,-1)."""
    xi = np.asarray(xi, dtype=float)
    eta = np.asarray(eta, dtype=float)
    dxi = 0.25 * np.stack([-(1 - eta), (1 - eta), (1 + eta), -(1 + eta)], -1)
    deta = 0.25 * np.stack([-(1 - xi), -(1 + xi), (1 + xi), (1 - xi)], -1)
    return dxi, deta


def _jacobian_at(xy, xi, eta):
    """(M, K, 2, 2) d(x,y)/d(xi,eta) at reference points (xi[k], eta[k])."""
    dxi, deta = _shape_derivs(xi, eta)
    J = np.empty((xy.shape[0], len(xi), 2, 2))
    J[..., 0, 0] = xy[:, :, 0] @ dxi.T
    J[..., 1, 0] = xy[:, :, 1] @ dxi.T
    J[..., 0, 1] = xy[:, :, 0] @ deta.T
    J[..., 1, 1] = xy[:, :, 1] @ deta.T
    return J


def build_mesh(nodes, elements, boundary, periodic_pairs=()) -> Mesh:
    """Face matching by shared corner pairs; see module docstring."""
    nodes = np.asarray(nodes, dtype=float).reshape(-1, 2)
    elements = np.asarray(elements, dtype=np.int64).reshape(-1, 4)
    if elements.size and (elements.min() < 0 or elements.max() >= len(nodes)):
        raise MeshError("element references a node index out of range")
    xy = nodes[elements]
    cxi = np.array([-1.0, 1.0, 1.0, -1.0])
    ceta = np.array([-1.0, -1.0, 1.0, 1.0])
    J = _jacobian_at(xy, cxi, ceta)
    det = J[..., 0, 0] * J[..., 1, 1] - J[..., 0, 1] * J[..., 1, 0]
    bad = np.nonzero((det <= 0.0).any(axis=1))[0]
    if bad.size:
        raise MeshError(f"element {bad[0]} has non-positive mapping Jacobian")

    pending = {}
    interior = []
    for e, corner in enumerate(elements.tolist()):
        for f, (i, j) in enumerate(FACE_NODES):
            a, b = corner[i], corner[j]
            key = (a, b) if a < b else (b, a)
            hit = pending.pop(key, None)
            if hit is None:
                pending[key] = (e, f, a, b)
            else:
                eL, fL, aL, bL = hit
                interior.append((eL, fL, e, f, int(aL == b and bL == a)))
    used = set()
    for eL, fL, eR, fR in periodic_pairs:
        interior.append((int(eL), int(fL), int(eR), int(fR), 1))
        used.update({(int(eL), int(fL)), (int(eR), int(fR))})

    bnd = []
    for e, f, _, _ in pending.values():
        if (e, f) in used:
            continue
        tag = boundary.get((e, f))
        if tag is None:
            raise MeshError(f"face {f} of element {e} has no neighbor and no boundary tag")
        if tag not in BOUNDARY_TAGS:
            raise MeshError(f"unknown boundary tag {tag!r}")
        bnd.append((e, f, tag))
    bnd.sort(key=lambda r: (r[0], r[1]))
    bnd_arr = np.array([(e, f) for e, f, _ in bnd], dtype=np.int64).reshape(-1, 2)
    tags = tuple(t for _, _, t in bnd)
    int_arr = np.array(sorted(interior), dtype=np.int64).reshape(-1, 5)
    return Mesh(nodes, elements, int_arr, bnd_arr, tags)


def generate_box(nx, ny, Lx, Ly, periodic=False, tag="far-field") -> Mesh:
    """Uniform nx x ny grid on [0,Lx]x[0,Ly]; element e = j*nx + i."""
    if nx < 1 or ny < 1:
        raise ValueError("nx and ny must be >= 1")
    X, Y = np.meshgrid(np.linspace(0.0, Lx, nx + 1),
                       np.linspace(0.0, Ly, ny + 1))
    nodes = np.stack([X.ravel(), Y.ravel()], axis=1)
    jj, ii = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    base = (jj * (nx + 1) + ii).ravel()
    elements = np.stack([base, base + 1, base + nx + 2, base + nx + 1], axis=1)
    eid = lambda i, j: j * nx + i
    boundary, pairs = {}, []
    if periodic:
        pairs += [(eid(nx - 1, j), 1, eid(0, j), 3) for j in range(ny)]
        pairs += [(eid(i, ny - 1), 2, eid(i, 0), 0) for i in range(nx)]
    else:
        for i in range(nx):
            boundary[(eid(i, 0), 0)] = tag
            boundary[(eid(i, ny - 1), 2)] = tag
        for j in range(ny):
            boundary[(eid(nx - 1, j), 1)] = tag
            boundary[(eid(0, j), 3)] = tag
    return build_mesh(nodes, elements, boundary, pairs)


def generate_channel(nx, ny, Lx, y_nodes, bottom="wall-adiabatic",
                     top="wall-slip") -> Mesh:
    """x-periodic channel on [0,Lx] x [y_nodes[0], y_nodes[-1]] with the
    given (possibly stretched) wall-normal node distribution; used for
    BASELINE config 4 via build_mesh + periodic pairs."""
    y_nodes = np.asarray(y_nodes, dtype=float)
    if len(y_nodes) != ny + 1:
        raise ValueError("need ny + 1 wall-normal node coordinates")
    X, Y = np.meshgrid(np.linspace(0.0, Lx, nx + 1), y_nodes)
    nodes = np.stack([X.ravel(), Y.ravel()], axis=1)
    jj, ii = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    base = (jj * (nx + 1) + ii).ravel()
    elements = np.stack([base, base + 1, base + nx + 2, base + nx + 1], axis=1)
    eid = lambda i, j: j * nx + i
    boundary = {}
    for i in range(nx):
        boundary[(eid(i, 0), 0)] = bottom
        boundary[(eid(i, ny - 1), 2)] = top
    pairs = [(eid(nx - 1, j), 1, eid(0, j), 3) for j in range(ny)]
    return build_mesh(nodes, elements, boundary, pairs)


def generate_cylinder_omesh(n_circ, n_rad, r_wall, r_far, stretch,
                            wall_tag="wall-adiabatic") -> Mesh:
    """O-grid; element (i, k) = k*n_circ + i, face 3 on the wall."""
    if n_circ < 8 or n_circ % 2:
        raise ValueError("n_circ must be an even number >= 8")
    if n_rad < 2:
        raise ValueError("n_rad must be >= 2")
    if r_far <= r_wall or r_wall <= 0:
        raise ValueError("need 0 < r_wall < r_far")
    if stretch < 1.0:
        raise ValueError("stretch must be >= 1")
    h0 = first_layer_height(n_rad, r_wall, r_far, stretch)
    if h0 <= 0.0:
        raise ValueError("first-layer height must be positive")
    layers = h0 * stretch ** np.arange(n_rad)
    radii = r_wall + np.concatenate(([0.0], np.cumsum(layers)))
    radii[-1] = r_far
    theta = 2.0 * np.pi * np.arange(n_circ) / n_circ
    R, T = np.meshgrid(radii, theta, indexing="ij")
    nodes = np.stack([(R * np.cos(T)).ravel(), (R * np.sin(T)).ravel()], 1)
    node = lambda i, k: k * n_circ + (i % n_circ)
    elements = np.array([(node(i, k), node(i, k + 1), node(i + 1, k + 1),
                          node(i + 1, k))
                         for k in range(n_rad) for i in range(n_circ)])
    boundary = {}
    for i in range(n_circ):
        boundary[(i, 3)] = wall_tag
        boundary[((n_rad - 1) * n_circ + i, 1)] = "far-field"
    return build_mesh(nodes, elements, boundary)


def first_layer_height(n_rad, r_wall, r_far, stretch) -> float:
    span = r_far - r_wall
    if stretch == 1.0:
        return span / n_rad
    return span * (stretch - 1.0) / (stretch ** n_rad - 1.0)


@dataclass(frozen=True)
class ElementGeometry:
    """Metrics at the degree-p points, layout as the reference's
    ElementGeometry (mesh.py:322-348)."""

    degree: int
    jac: np.ndarray
    det: np.ndarray
    inv: np.ndarray
    face_normals: np.ndarray
    face_jac: np.ndarray
    face_det: np.ndarray
    face_jac_cols: np.ndarray
    h_min: np.ndarray

    @property
    def n(self) -> int:
        return self.degree + 1


def element_geometry(mesh: Mesh, p: int, elems=None) -> ElementGeometry:
    elems = np.arange(mesh.n_elements) if elems is None else np.asarray(elems, np.int64)
    xy = mesh.nodes[mesh.elements[elems]]
    pts = basis(p).points
    n = p + 1
    eta_g, xi_g = np.meshgrid(pts, pts, indexing="ij")
    J = _jacobian_at(xy, xi_g.ravel(), eta_g.ravel()).reshape(len(elems), n, n, 2, 2)
    det = J[..., 0, 0] * J[..., 1, 1] - J[..., 0, 1] * J[..., 1, 0]
    if (det <= 0.0).any():
        m = int(elems[np.nonzero((det <= 0.0).any(axis=(1, 2)))[0][0]])
        raise MeshError(f"element {m} has non-positive mapping Jacobian")
    inv = np.empty_like(J)
    inv[..., 0, 0] = J[..., 1, 1] / det
    inv[..., 0, 1] = -J[..., 0, 1] / det
    inv[..., 1, 0] = -J[..., 1, 0] / det
    inv[..., 1, 1] = J[..., 0, 0] / det
    edges = np.roll(xy, -1, axis=1) - xy
    elen = np.sqrt((edges * edges).sum(axis=2))
    normals = np.stack([edges[..., 1], -edges[..., 0]], axis=-1) / elen[..., None]
    ones = np.ones(n)
    fxi = np.concatenate([pts, ones, pts[::-1], -ones])
    feta = np.concatenate([-ones, pts, ones, pts[::-1]])
    Jf = _jacobian_at(xy, fxi, feta).reshape(len(elems), 4, n, 2, 2)
    detf = Jf[..., 0, 0] * Jf[..., 1, 1] - Jf[..., 0, 1] * Jf[..., 1, 0]
    return ElementGeometry(p, J, det, inv, normals, 0.5 * elen, detf, Jf,
                           elen.min(axis=1))


def solution_point_coords(mesh: Mesh, p: int, elems=None) -> np.ndarray:
    """(M, n, n, 2) physical coordinates of the solution points."""
    elems = np.arange(mesh.n_elements) if elems is None else np.asarray(elems, np.int64)
    pts = basis(p).points
    eta_g, xi_g = np.meshgrid(pts, pts, indexing="ij")
    xi, eta = xi_g.ravel(), eta_g.ravel()
    N = 0.25 * np.stack([(1 - xi) * (1 - eta), (1 + xi) * (1 - eta),
                         (1 + xi) * (1 + eta), (1 - xi) * (1 + eta)], -1)
    xy = np.einsum("ka,maj->mkj", N, mesh.nodes[mesh.elements[elems]])
    n = p + 1
    return xy.reshape(len(elems), n, n, 2)


# ---------------------------------------------------------------------------
# device packing

def face_links(mesh: Mesh):
    """Per (element, face) neighbour link table.

    Returns int64 (M, 4, 4) with columns (neighbour element, neighbour
    face, rev, is_left) and int32 (M, 4) boundary tag code (-1 for
    interior faces).  is_left marks the side that owns the reference's
    flux evaluation (interior_faces column 0, spatial.py:521-526).
    """
    M = mesh.n_elements
    link = np.full((M, 4, 4), -1, dtype=np.int64)
    tag = np.full((M, 4), -1, dtype=np.int32)
    for eL, fL, eR, fR, rev in mesh.interior_faces.tolist():
        link[eL, fL] = (eR, fR, rev, 1)
        link[eR, fR] = (eL, fL, rev, 0)
    for (e, f), t in zip(mesh.boundary_faces.tolist(), mesh.boundary_tags):
        tag[e, f] = TAG_CODE[t]
        link[e, f] = (-1, 0, 0, 1)
    if (link[..., 0] < 0).sum() != len(mesh.boundary_tags):
        raise MeshError("face link table incomplete")
    return link, tag


def pack_geometry(mesh: Mesh) -> np.ndarray:
    """(M, 20) float64 per-element record the kernels read.

    [0:8]   bilinear metric coefficients: x_xi = c0 + c1*eta,
            y_xi = c2 + c3*eta, x_eta = c4 + c5*xi, y_eta = c6 + c7*xi
            (the Q1 map of mesh.py:309-318 is affine per direction)
    [8:16]  outward unit normals (nx, ny) of faces 0..3 (mesh.py:382-385)
    [16:20] face_jac = |edge| / 2 of faces 0..3
    """
    xy = mesh.nodes[mesh.elements]
    x, y = xy[..., 0], xy[..., 1]
    out = np.empty((mesh.n_elements, 20))
    for k, c in enumerate((x, y)):
        s01, s32 = c[:, 1] - c[:, 0], c[:, 2] - c[:, 3]
        s30, s21 = c[:, 3] - c[:, 0], c[:, 2] - c[:, 1]
        out[:, 2 * k] = 0.25 * (s01 + s32)
        out[:, 2 * k + 1] = 0.25 * (s32 - s01)
        out[:, 4 + 2 * k] = 0.25 * (s30 + s21)
        out[:, 4 + 2 * k + 1] = 0.25 * (s21 - s30)
    g = element_geometry(mesh, 0)
    out[:, 8:16] = g.face_normals.reshape(-1, 8)
    out[:, 16:20] = g.face_jac
    return out
