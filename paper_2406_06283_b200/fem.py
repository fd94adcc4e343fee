"""Setup phase, part 1: structured P1 mesh, FE space and global forms.

Host-side restatement of the reference's setup so that the GPU solve phase
can be fed on a box where the reference package is absent.  The objects carry
the same attribute names as the reference dataclasses, so either set of
objects can be handed to :func:`paper_2406_06283_b200.factorize`.

Reference behaviour followed:
  * mesh:      pkg/src/helmdd/mesh.py:68-121   (2 n^2 right triangles, diagonal
                                               lower-left -> upper-right,
                                               row-major vertices)
  * FE space:  mesh.py:124-134                 (interior vertices, lexicographic)
  * coefficient: assembly.py:23-63             (+ a per-cell random field, the
                                               SURVEY D8 extension)
  * forms:     assembly.py:90-145              (exact P1 element matrices,
                                               COO->CSR, B = A - k^2 S,
                                               D_k = A + k^2 S)
  * load:      assembly.py:148-168             (edge-midpoint rule)
  * local forms: assembly.py:171-194
"""

from dataclasses import dataclass

import numpy as np
from scipy import sparse

_MASS_REF = np.array([[2.0, 1.0, 1.0], [1.0, 2.0, 1.0], [1.0, 1.0, 2.0]]) / 12.0


@dataclass(frozen=True)
class Mesh:
    n_per_side: int
    vertices: np.ndarray
    triangles: np.ndarray
    h: float
    boundary_vertex_flags: np.ndarray
    incidence: sparse.csr_matrix

    @property
    def n_vertices(self):
        return self.vertices.shape[0]

    @property
    def n_triangles(self):
        return self.triangles.shape[0]

    @property
    def vertex_degree(self):
        return np.bincount(self.triangles.ravel(), minlength=self.n_vertices)


@dataclass(frozen=True)
class FeSpace:
    n_dofs: int
    dof_of_vertex: np.ndarray
    vertex_of_dof: np.ndarray


def build_unit_square_mesh(n_per_side):
    """Uniform n x n cell grid of [0,1]^2, two triangles per cell (mesh.py:68-121).

    Cell (cx, cy) owns triangles 2*(cy*n+cx) (lower: v00,v10,v11) and +1
    (upper: v00,v11,v01); vertices are numbered row-major, y outer.
    """
    n = int(n_per_side)
    if n < 2:
        raise ValueError("n_per_side must be >= 2, got %r" % (n_per_side,))
    coords = np.arange(n + 1, dtype=float) / n
    vy, vx = np.divmod(np.arange((n + 1) * (n + 1)), n + 1)
    vertices = np.column_stack([coords[vx], coords[vy]])
    cy, cx = np.divmod(np.arange(n * n), n)
    base = cy * (n + 1) + cx
    tri = np.empty((2 * n * n, 3), dtype=np.int64)
    tri[0::2, 0] = base
    tri[0::2, 1] = base + 1
    tri[0::2, 2] = base + n + 2
    tri[1::2, 0] = base
    tri[1::2, 1] = base + n + 2
    tri[1::2, 2] = base + n + 1
    pts = vertices[tri]
    edges = np.stack([pts[:, 1] - pts[:, 0], pts[:, 2] - pts[:, 1], pts[:, 0] - pts[:, 2]], axis=1)
    h = float(np.sqrt((edges**2).sum(axis=2)).max())
    del pts, edges
    boundary = (vx == 0) | (vx == n) | (vy == 0) | (vy == n)
    nt = tri.shape[0]
    incidence = sparse.csr_matrix(
        (np.ones(3 * nt), tri.ravel(), np.arange(0, 3 * nt + 1, 3)),
        shape=(nt, vertices.shape[0]),
    )
    return Mesh(n, vertices, tri, h, boundary, incidence)


def build_fe_space(mesh):
    """Dofs = interior vertices in lexicographic vertex order (mesh.py:124-134)."""
    vertex_of_dof = np.flatnonzero(~mesh.boundary_vertex_flags)
    dof_of_vertex = np.full(mesh.n_vertices, -1, dtype=np.int64)
    dof_of_vertex[vertex_of_dof] = np.arange(vertex_of_dof.size)
    return FeSpace(int(vertex_of_dof.size), dof_of_vertex, vertex_of_dof)


def triangle_areas(mesh):
    p = mesh.vertices[mesh.triangles]
    e1 = p[:, 1] - p[:, 0]
    e2 = p[:, 2] - p[:, 0]
    return 0.5 * (e1[:, 0] * e2[:, 1] - e1[:, 1] * e2[:, 0])


@dataclass(frozen=True)
class CoefficientField:
    kind: str
    contrast: float
    per_element_value: np.ndarray


def _cell_index(mesh, blocks):
    cent = mesh.vertices[mesh.triangles].mean(axis=1)
    nb = int(blocks)
    bx = np.minimum((cent[:, 0] * nb).astype(int), nb - 1)
    by = np.minimum((cent[:, 1] * nb).astype(int), nb - 1)
    return bx, by


def coefficient_field(mesh, kind="constant", contrast=1.0, blocks=4):
    """Constant / checkerboard / channels fields (assembly.py:35-63)."""
    contrast = float(contrast)
    if contrast < 1.0:
        raise ValueError("contrast must be >= 1, got %g" % contrast)
    if int(blocks) < 1:
        raise ValueError("blocks must be >= 1")
    bx, by = _cell_index(mesh, blocks)
    if kind == "constant":
        if contrast != 1.0:
            raise ValueError("constant coefficient requires contrast == 1")
        vals = np.ones(mesh.n_triangles)
    elif kind == "checkerboard":
        vals = np.where((bx + by) % 2 == 1, contrast, 1.0)
    elif kind == "channels":
        vals = np.where(by % 2 == 1, contrast, 1.0)
    else:
        raise ValueError("unknown coefficient kind %r" % (kind,))
    return CoefficientField(kind, contrast, vals)


def loguniform_cell_field(mesh, cells, lo, hi, seed):
    """Piecewise-constant a(x) on a cells x cells grid, log-uniform in [lo, hi].

    SURVEY D8: the BASELINE configs 3/5 ask for this field, which the
    reference's coefficient_field does not know; triangles are mapped to
    their cell by centroid exactly as assembly.py:46-51 does.
    """
    rng = np.random.default_rng(seed)
    table = np.exp(rng.uniform(np.log(lo), np.log(hi), size=(cells, cells)))
    bx, by = _cell_index(mesh, cells)
    vals = table[by, bx]
    return CoefficientField("loguniform_cells", float(hi / lo), vals)


@dataclass(frozen=True)
class AssembledForms:
    k: float
    stiffness: sparse.csr_matrix
    mass: sparse.csr_matrix
    helmholtz: sparse.csr_matrix
    dk: sparse.csr_matrix
    elem_stiffness: np.ndarray
    elem_mass: np.ndarray
    tri_dofs: np.ndarray

    @property
    def n_dofs(self):
        return self.stiffness.shape[0]


def element_matrices(mesh, coeff):
    """Exact P1 stiffness (with coefficient) and mass per triangle (assembly.py:90-109)."""
    p = mesh.vertices[mesh.triangles]
    x, y = p[:, :, 0], p[:, :, 1]
    det = (x[:, 1] - x[:, 0]) * (y[:, 2] - y[:, 0]) - (x[:, 2] - x[:, 0]) * (y[:, 1] - y[:, 0])
    area = 0.5 * det
    # gradient of the barycentric function of vertex a: perp of the opposite edge
    gx = np.stack([y[:, 1] - y[:, 2], y[:, 2] - y[:, 0], y[:, 0] - y[:, 1]], axis=1)
    gy = np.stack([x[:, 2] - x[:, 1], x[:, 0] - x[:, 2], x[:, 1] - x[:, 0]], axis=1)
    grads = np.stack([gx, gy], axis=2) / det[:, None, None]
    # a * area * grad_a . grad_b, contracted with einsum so the rounding is
    # that of assembly.py:107 (bitwise-identical forms)
    stiff = np.einsum("t,tad,tbd->tab", coeff.per_element_value * area, grads, grads)
    mass = area[:, None, None] * _MASS_REF[None, :, :]
    return stiff, mass


def _scatter(elem, tri_dofs, n):
    rows = np.repeat(tri_dofs, 3, axis=1).ravel()
    cols = np.tile(tri_dofs, (1, 3)).ravel()
    keep = (rows >= 0) & (cols >= 0)
    return sparse.coo_matrix((elem.ravel()[keep], (rows[keep], cols[keep])), shape=(n, n)).tocsr()


def assemble_forms(mesh, space, coeff, k):
    """A, S, B = A - k^2 S and D_k = A + k^2 S over the interior dofs (assembly.py:123-145)."""
    if k <= 0:
        raise ValueError("wavenumber k must be positive, got %g" % k)
    if coeff.per_element_value.shape[0] != mesh.n_triangles:
        raise ValueError("coefficient field does not cover every triangle")
    stiff, mass = element_matrices(mesh, coeff)
    tri_dofs = space.dof_of_vertex[mesh.triangles]
    A = _scatter(stiff, tri_dofs, space.n_dofs)
    S = _scatter(mass, tri_dofs, space.n_dofs)
    k2 = float(k) * float(k)
    return AssembledForms(
        k=float(k),
        stiffness=A,
        mass=S,
        helmholtz=(A - k2 * S).tocsr(),
        dk=(A + k2 * S).tocsr(),
        elem_stiffness=stiff,
        elem_mass=mass,
        tri_dofs=tri_dofs,
    )


def assemble_rhs(mesh, space, f):
    """Load vector (f, phi_i) by the edge-midpoint rule (assembly.py:148-168)."""
    p = mesh.vertices[mesh.triangles]
    area = triangle_areas(mesh)
    mids = [0.5 * (p[:, 0] + p[:, 1]), 0.5 * (p[:, 1] + p[:, 2]), 0.5 * (p[:, 2] + p[:, 0])]
    f01, f12, f20 = (np.asarray(f(m[:, 0], m[:, 1]), dtype=float) for m in mids)
    contrib = np.stack([f01 + f20, f01 + f12, f12 + f20], axis=1) * (area / 6.0)[:, None]
    tri_dofs = space.dof_of_vertex[mesh.triangles]
    keep = tri_dofs >= 0
    return np.bincount(tri_dofs[keep], weights=contrib[keep], minlength=space.n_dofs).astype(float)


def rhs_function(spec, h):
    """The reference CLI's rhs specs: 'constant' and 'gaussian[:cx,cy,w]' (cli.py:186-201)."""
    spec = spec.strip()
    if spec == "constant":
        return lambda x, y: np.ones_like(x)
    if spec.startswith("gaussian"):
        cx, cy, width = 0.5, 0.5, 2.0 * h
        if ":" in spec:
            parts = spec.split(":", 1)[1].split(",")
            if len(parts) != 3:
                raise ValueError("gaussian rhs wants 'gaussian:cx,cy,width'")
            cx, cy = float(parts[0]), float(parts[1])
            width = 2.0 * h if parts[2] == "auto" else float(parts[2])
        return lambda x, y: np.exp(-((x - cx) ** 2 + (y - cy) ** 2) / (2.0 * width**2))
    raise ValueError("unknown rhs spec %r" % (spec,))


def local_forms_sparse(forms, elements, dofs):
    """Subassembled stiffness and mass over an element subset, as CSR over ``dofs``.

    Same matrices as assembly.py:171-194 (natural coupling on the internal
    boundary) but sparse, so large subdomains stay cheap.
    """
    dofs = np.asarray(dofs)
    lookup = np.full(forms.n_dofs, -1, dtype=np.int64)
    lookup[dofs] = np.arange(dofs.size)
    td = forms.tri_dofs[elements]
    loc = np.where(td >= 0, lookup[td], -1)
    if np.any((td >= 0) & (loc < 0)):
        raise ValueError("dof list does not cover all dofs active on the elements")
    rows = np.repeat(loc, 3, axis=1).ravel()
    cols = np.tile(loc, (1, 3)).ravel()
    keep = (rows >= 0) & (cols >= 0)
    shape = (dofs.size, dofs.size)
    A = sparse.coo_matrix((forms.elem_stiffness[elements].ravel()[keep], (rows[keep], cols[keep])), shape=shape).tocsr()
    S = sparse.coo_matrix((forms.elem_mass[elements].ravel()[keep], (rows[keep], cols[keep])), shape=shape).tocsr()
    return A, S


def assemble_local_forms(forms, elements, dofs):
    """Dense local stiffness and mass, accumulated element by element in
    element order like assembly.py:171-194 (so the values match bitwise)."""
    dofs = np.asarray(dofs)
    lookup = np.full(forms.n_dofs, -1, dtype=np.int64)
    lookup[dofs] = np.arange(dofs.size)
    td = forms.tri_dofs[elements]
    loc = np.where(td >= 0, lookup[td], -1)
    if np.any((td >= 0) & (loc < 0)):
        raise ValueError("dof list does not cover all dofs active on the elements")
    rows = np.repeat(loc, 3, axis=1).ravel()
    cols = np.tile(loc, (1, 3)).ravel()
    keep = (rows >= 0) & (cols >= 0)
    A = np.zeros((dofs.size, dofs.size))
    S = np.zeros((dofs.size, dofs.size))
    np.add.at(A, (rows[keep], cols[keep]), forms.elem_stiffness[elements].ravel()[keep])
    np.add.at(S, (rows[keep], cols[keep]), forms.elem_mass[elements].ravel()[keep])
    return A, S
