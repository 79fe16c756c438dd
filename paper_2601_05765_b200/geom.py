"""Host-side geometry: planes, convex polytopes and the packed kernel layout.

This mirrors the part of the reference's ``potflow.geom`` that feeds the hot
path (/root/reference/pkg/src/potflow/geom.py):

* ``Plane`` / ``Facet`` / ``ConvexCell``          geom.py:62-166
* facet tags (site j >= 0, domain face -(k+1))    geom.py:44-59
* ``init_cell_from_domain`` / ``box_domain``      geom.py:392-475
* ``pack_cell`` / ``unpack_cell``                 geom.py:353-385
* ``cell_volume_convex`` / ``cell_centroid_convex`` geom.py:506-537

Domain set-up runs once per scene on the host; everything per-cell runs on
the B200 (see ``_kernels`` / ``restricted``).  The domain pack produced here
is bit-identical to the reference's (tests/test_geom_host.py pins it against
tests/golden fixtures produced by the reference).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

DEFAULT_REL_TOL = 1e-9

# packed-layout capacities of the reference kernels (_kernels.py:24-27)
MAX_V, MAX_F, MAX_L, MAX_P = 512, 160, 2048, 256


class GeomError(Exception):
    """Base class for geometry errors."""


class UnboundedDomain(GeomError):
    pass


class EmptyDomain(GeomError):
    pass


class OpenLoop(GeomError):
    pass


def tag_site(j: int) -> int:
    return int(j)


def tag_domain(k: int) -> int:
    return -(int(k) + 1)


def tag_is_site(tag: int) -> bool:
    return tag >= 0


def tag_index(tag: int) -> int:
    return tag if tag >= 0 else -tag - 1


def perp_basis(n) -> tuple[np.ndarray, np.ndarray]:
    """Canonical in-plane frame (e1, e2) of a unit normal (_kernels.py:59-80)."""
    nx, ny, nz = float(n[0]), float(n[1]), float(n[2])
    a = (abs(nx), abs(ny), abs(nz))
    if a[0] <= a[1] and a[0] <= a[2]:
        u = (1.0, 0.0, 0.0)
    elif a[1] <= a[2]:
        u = (0.0, 1.0, 0.0)
    else:
        u = (0.0, 0.0, 1.0)
    e1 = [u[1] * nz - u[2] * ny, u[2] * nx - u[0] * nz, u[0] * ny - u[1] * nx]
    inv = 1.0 / math.sqrt(e1[0] * e1[0] + e1[1] * e1[1] + e1[2] * e1[2])
    e1 = [e1[0] * inv, e1[1] * inv, e1[2] * inv]
    e2 = [ny * e1[2] - nz * e1[1], nz * e1[0] - nx * e1[2], nx * e1[1] - ny * e1[0]]
    return np.array(e1), np.array(e2)


@dataclass
class Plane:
    """Oriented plane n.x = d, inside is n.x <= d; n is normalised on entry."""

    n: np.ndarray
    d: float

    def __post_init__(self):
        self.n = np.asarray(self.n, dtype=np.float64)
        norm = float(np.linalg.norm(self.n))
        if not math.isfinite(norm) or abs(norm - 1.0) > 1e-9:
            if not math.isfinite(norm) or norm <= 0.0:
                raise GeomError("plane normal must be a nonzero finite vector")
            self.n = self.n / norm
            self.d = float(self.d) / norm
        self.d = float(self.d)

    @classmethod
    def from_point_normal(cls, point, normal) -> "Plane":
        normal = np.asarray(normal, dtype=np.float64)
        normal = normal / np.linalg.norm(normal)
        return cls(normal, float(np.dot(normal, point)))

    def signed_distance(self, x) -> float:
        return float(np.dot(self.n, x) - self.d)


@dataclass
class Facet:
    plane: Plane
    loop: np.ndarray  # vertex indices, CCW seen from outside
    tag: int

    def __post_init__(self):
        self.loop = np.asarray(self.loop, dtype=np.int64)


@dataclass
class ConvexCell:
    vertices: np.ndarray
    facets: list

    def __post_init__(self):
        self.vertices = np.asarray(self.vertices, dtype=np.float64).reshape(-1, 3)

    @property
    def n_vertices(self) -> int:
        return self.vertices.shape[0]

    @property
    def n_facets(self) -> int:
        return len(self.facets)

    def n_edges(self) -> int:
        return sum(len(f.loop) for f in self.facets) // 2

    def bbox(self):
        return self.vertices.min(axis=0), self.vertices.max(axis=0)

    def diagonal(self) -> float:
        lo, hi = self.bbox()
        return float(np.linalg.norm(hi - lo))

    def contains(self, x, tol: float = 0.0) -> bool:
        return all(f.plane.signed_distance(x) <= tol for f in self.facets)

    def validate(self, tol: float | None = None) -> None:
        """Euler / edge-twice / on-plane invariants (geom.py:134-165)."""
        if tol is None:
            tol = DEFAULT_REL_TOL * max(self.diagonal(), 1.0)
        edges: dict = {}
        incident = np.zeros(self.n_vertices, dtype=int)
        for f in self.facets:
            if len(f.loop) < 3:
                raise GeomError("facet loop with fewer than 3 vertices")
            ring = np.roll(f.loop, -1)
            for a, b in zip(f.loop.tolist(), ring.tolist()):
                key = (a, b) if a < b else (b, a)
                edges[key] = edges.get(key, 0) + 1
            dist = self.vertices @ f.plane.n - f.plane.d
            if np.any(dist > tol):
                raise GeomError("vertex outside a facet halfspace")
            on = np.abs(dist) <= tol
            incident[on] += 1
            if not np.all(on[f.loop]):
                raise GeomError("loop vertex not on its facet plane")
        bad = [k for k, c in edges.items() if c != 2]
        if bad:
            raise GeomError(f"edge {bad[0]} not shared by exactly 2 facets")
        if self.n_vertices - len(edges) + self.n_facets != 2:
            raise GeomError("Euler characteristic violated")
        if np.any(incident < 3):
            raise GeomError("vertex incident to fewer than 3 facet planes")


def init_cell_from_domain(halfspaces: list, tol: float | None = None) -> ConvexCell:
    """Polytope of an intersection of halfspaces (geom.py:392-460).

    Vertices come from every feasible plane triple (first occurrence kept);
    each non-redundant plane becomes a facet tagged ``tag_domain(k)`` whose
    loop is ordered by (angle about the vertex mean in the plane's canonical
    frame, vertex index).
    """
    m = len(halfspaces)
    if m < 4:
        raise UnboundedDomain("fewer than 4 halfspaces cannot bound a polytope")
    N = np.array([h.n for h in halfspaces])
    d = np.array([h.d for h in halfspaces])
    from scipy.optimize import linprog

    for sign in (1.0, -1.0):
        for axis in range(3):
            c = np.zeros(3)
            c[axis] = -sign
            res = linprog(c, A_ub=N, b_ub=d, bounds=[(None, None)] * 3, method="highs")
            if res.status == 3:
                raise UnboundedDomain("halfspace intersection is unbounded")
            if res.status == 2:
                raise EmptyDomain("halfspace intersection is empty")
    cand = []
    for i in range(m):
        for j in range(i + 1, m):
            for k in range(j + 1, m):
                A = np.array([N[i], N[j], N[k]])
                if abs(np.linalg.det(A)) < 1e-12:
                    continue
                cand.append(np.linalg.solve(A, np.array([d[i], d[j], d[k]])))
    if not cand:
        raise EmptyDomain("no plane triples intersect")
    cand = np.array(cand)
    scale = float(np.max(np.ptp(cand, axis=0))) if len(cand) > 1 else 1.0
    if tol is None:
        tol = DEFAULT_REL_TOL * max(scale, 1.0)
    feas = cand[np.all(cand @ N.T - d <= tol, axis=1)]
    if len(feas) == 0:
        raise EmptyDomain("halfspace intersection is empty")
    verts: list = []
    for p in feas:
        if all(np.linalg.norm(p - q) > tol for q in verts):
            verts.append(p)
    V = np.array(verts)
    if len(V) < 4:
        raise EmptyDomain("degenerate (lower-dimensional) intersection")
    facets = []
    for k in range(m):
        on = np.nonzero(np.abs(V @ N[k] - d[k]) <= tol)[0]
        if len(on) < 3:
            continue
        e1, e2 = perp_basis(N[k])
        ctr = V[on].mean(axis=0)
        ang = np.arctan2((V[on] - ctr) @ e2, (V[on] - ctr) @ e1)
        facets.append(Facet(Plane(N[k].copy(), float(d[k])), on[np.lexsort((on, ang))],
                            tag_domain(k)))
    cell = ConvexCell(V, facets)
    cell.validate(tol)
    return cell


def box_domain(lo, hi) -> ConvexCell:
    """Axis-aligned box, faces ordered -x +x -y +y -z +z (geom.py:463-475)."""
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    planes = []
    for axis in range(3):
        e = np.zeros(3)
        e[axis] = 1.0
        planes.append(Plane(-e, -lo[axis]))
        planes.append(Plane(e.copy(), hi[axis]))
    return init_cell_from_domain(planes)


def pack_cell(cell: ConvexCell):
    """ConvexCell -> reference packed arrays (geom.py:353-375)."""
    nv, nf = cell.n_vertices, cell.n_facets
    nl = sum(len(f.loop) for f in cell.facets)
    if nv > MAX_V or nf > MAX_F or nl > MAX_L:
        raise GeomError("cell exceeds kernel buffer capacity")
    verts = np.zeros((MAX_V, 3))
    planes = np.zeros((MAX_F, 4))
    tags = np.zeros(MAX_F, dtype=np.int64)
    lp = np.zeros(MAX_F + 1, dtype=np.int64)
    lv = np.zeros(MAX_L, dtype=np.int64)
    verts[:nv] = cell.vertices
    offs = np.cumsum([0] + [len(f.loop) for f in cell.facets])
    for f, fac in enumerate(cell.facets):
        planes[f, :3] = fac.plane.n
        planes[f, 3] = fac.plane.d
        tags[f] = fac.tag
        lv[offs[f]:offs[f + 1]] = fac.loop
    lp[:nf + 1] = offs
    return verts, np.array([nv, nf, nl], dtype=np.int64), planes, tags, lp, lv


def unpack_cell(verts, cnt, planes, tags, lp, lv) -> ConvexCell:
    """Packed arrays -> ConvexCell (geom.py:378-385)."""
    nv, nf = int(cnt[0]), int(cnt[1])
    facets = [Facet(Plane(np.array(planes[f, :3], dtype=np.float64), float(planes[f, 3])),
                    np.array(lv[lp[f]:lp[f + 1]], dtype=np.int64), int(tags[f]))
              for f in range(nf)]
    return ConvexCell(np.array(verts[:nv], dtype=np.float64), facets)


def _fan(cell: ConvexCell):
    apex = cell.vertices.mean(axis=0)
    for f in cell.facets:
        p0 = cell.vertices[f.loop[0]]
        for k in range(1, len(f.loop) - 1):
            p1 = cell.vertices[f.loop[k]]
            p2 = cell.vertices[f.loop[k + 1]]
            yield apex, p0, p1, p2, np.dot(np.cross(p1 - p0, p2 - p0), p0 - apex)


def cell_volume_convex(cell: ConvexCell) -> float:
    """Polytope volume from apex-fan tetrahedra (geom.py:506-518)."""
    return abs(sum(v6 for *_, v6 in _fan(cell))) / 6.0


def cell_centroid_convex(cell: ConvexCell) -> np.ndarray:
    """Polytope volume centroid (geom.py:521-537)."""
    vol = 0.0
    mom = np.zeros(3)
    apex = cell.vertices.mean(axis=0)
    for a, p0, p1, p2, v6 in _fan(cell):
        vol += v6
        mom += v6 * (p0 + p1 + p2 + a)
    if vol == 0.0:
        return apex
    return mom / (4.0 * vol)
