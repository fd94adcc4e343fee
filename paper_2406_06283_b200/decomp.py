"""Setup phase, part 2: the nested two-level overlapping decomposition.

Restates pkg/src/helmdd/decomp.py:105-265 (build_two_level and its dof
bookkeeping) with identical results, but every subdomain is built inside a
local window of cells around its box instead of over the whole mesh: one
layer of vertex-adjacent extension grows a set by at most one cell in each
direction, so the window [box - layers, box + layers) contains the extended
set.  That turns the reference's O(N_sub * n_triangles) loop into
O(sum of window sizes), which is what makes the ~1M-dof configs tractable.

Index conventions follow the reference exactly: coarse subdomains ordered
(by outer, bx inner), fine pieces (py outer, px inner), ovdof/idof ascending,
pou = 1/multiplicity on interior dofs (decomp.py:251-265).
"""

from dataclasses import dataclass, field

import numpy as np
from scipy.spatial import ConvexHull, QhullError

from .errors import ConfigError


@dataclass(frozen=True)
class Subdomain:
    elements: np.ndarray
    ovdof: np.ndarray
    idof: np.ndarray
    idof_in_ov: np.ndarray
    pou: np.ndarray
    diameter: float
    n_triangles: int = field(default=0, repr=False)

    @property
    def element_mask(self):
        mask = np.zeros(self.n_triangles, dtype=bool)
        mask[self.elements] = True
        return mask


@dataclass(frozen=True)
class TwoLevelDecomposition:
    coarse: list
    fine: list
    coarse_multiplicity: np.ndarray
    fine_multiplicity: np.ndarray
    Lambda: int
    Hc: float
    Hf: float
    layers_c: int
    layers_f: int

    @property
    def n_coarse(self):
        return len(self.coarse)

    @property
    def fine_counts(self):
        return [len(fam) for fam in self.fine]

    def fine_flat(self):
        for i, fam in enumerate(self.fine):
            for j, sub in enumerate(fam):
                yield i, j, sub


class _Window:
    """Cells [x0, x1) x [y0, y1) of the global grid with local triangle/vertex maps."""

    def __init__(self, n, x0, x1, y0, y1):
        self.n = n
        self.x0, self.x1, self.y0, self.y1 = x0, x1, y0, y1
        wx, wy = x1 - x0, y1 - y0
        ly, lx = np.divmod(np.arange(wx * wy), wx)
        self.cell_x = np.repeat(lx + x0, 2)
        self.cell_y = np.repeat(ly + y0, 2)
        gcell = (ly + y0) * n + (lx + x0)
        self.gtri = np.empty(2 * wx * wy, dtype=np.int64)
        self.gtri[0::2] = 2 * gcell
        self.gtri[1::2] = 2 * gcell + 1
        # local vertex grid (wx+1) x (wy+1)
        base = ly * (wx + 1) + lx
        tri = np.empty((2 * wx * wy, 3), dtype=np.int64)
        tri[0::2] = np.column_stack([base, base + 1, base + wx + 2])
        tri[1::2] = np.column_stack([base, base + wx + 2, base + wx + 1])
        self.tri = tri
        vy, vx = np.divmod(np.arange((wx + 1) * (wy + 1)), wx + 1)
        self.gvert = (vy + y0) * (n + 1) + (vx + x0)

    def extend(self, mask, layers):
        if not mask.any():
            raise ValueError("cannot extend an empty element set")
        for _ in range(int(layers)):
            touched = np.zeros(self.gvert.size, dtype=bool)
            touched[self.tri[mask].ravel()] = True
            mask = touched[self.tri].any(axis=1)
        return mask


def _window_for_box(n, x0, x1, y0, y1, layers):
    return _Window(n, max(0, x0 - layers), min(n, x1 + layers), max(0, y0 - layers), min(n, y1 + layers))


def _dofs_of(win, mask, space, degree):
    count = np.bincount(win.tri[mask].ravel(), minlength=win.gvert.size)
    gv = win.gvert
    d_act = space.dof_of_vertex[gv[count > 0]]
    d_int = space.dof_of_vertex[gv[count == degree[gv]]]
    return np.sort(d_act[d_act >= 0]), np.sort(d_int[d_int >= 0]), gv[count > 0]


def _diameter(points):
    if points.shape[0] > 256:
        try:
            points = points[ConvexHull(points).vertices]
        except QhullError:
            pass
    diff = points[:, None, :] - points[None, :, :]
    return float(np.sqrt((diff**2).sum(axis=2)).max())


def build_two_level(mesh, space, coarse_m, fine_q, layers_c=1, layers_f=1):
    """M x M coarse boxes extended by layers_c, each split into q x q fine boxes
    extended by layers_f and clipped to the coarse subdomain (decomp.py:105-210)."""
    n = mesh.n_per_side
    M, q = int(coarse_m), int(fine_q)
    if M < 1 or n % M != 0:
        raise ConfigError("coarse_M=%d must divide n_per_side=%d" % (M, n))
    wc = n // M
    if q < 1 or wc % q != 0:
        raise ConfigError("fine_q=%d must divide n_per_side/coarse_M=%d" % (q, wc))
    if layers_c < 1 or layers_f < 1:
        raise ConfigError("both overlap layer counts must be >= 1")
    wf = wc // q
    degree = mesh.vertex_degree

    raw_coarse = []
    raw_fine = []
    for by in range(M):
        for bx in range(M):
            win = _window_for_box(n, bx * wc, (bx + 1) * wc, by * wc, (by + 1) * wc, layers_c)
            base = (
                (win.cell_x >= bx * wc) & (win.cell_x < (bx + 1) * wc)
                & (win.cell_y >= by * wc) & (win.cell_y < (by + 1) * wc)
            )
            ext = win.extend(base, layers_c)
            raw_coarse.append((win, ext))
            jx = np.clip((win.cell_x - bx * wc) // wf, 0, q - 1)
            jy = np.clip((win.cell_y - by * wc) // wf, 0, q - 1)
            fam = []
            for py in range(q):
                for px in range(q):
                    piece = ext & (jx == px) & (jy == py)
                    if not piece.any():
                        raise ConfigError(
                            "empty fine subdomain (%d, %d) in coarse box %d" % (px, py, len(raw_coarse) - 1)
                        )
                    fam.append(win.extend(piece, layers_f) & ext)
            raw_fine.append(fam)

    coarse_sets = [_dofs_of(win, m, space, degree) for win, m in raw_coarse]
    fine_sets = [[_dofs_of(win, m, space, degree) for m in fam] for (win, _), fam in zip(raw_coarse, raw_fine)]
    mu_c = np.zeros(space.n_dofs, dtype=np.int64)
    for _, idof, _ in coarse_sets:
        mu_c[idof] += 1
    mu_f = np.zeros(space.n_dofs, dtype=np.int64)
    for fam in fine_sets:
        for _, idof, _ in fam:
            mu_f[idof] += 1
    if np.any(mu_c < 1) or np.any(mu_f < 1):
        raise ConfigError("partition of unity does not cover every dof; increase the overlap layers")

    nt = mesh.n_triangles

    def make(win, mask, sets, mu):
        ovdof, idof, verts = sets
        pos = np.searchsorted(ovdof, idof)
        pou = np.zeros(ovdof.size)
        pou[pos] = 1.0 / mu[idof]
        return Subdomain(
            elements=np.sort(win.gtri[mask]),
            ovdof=ovdof,
            idof=idof,
            idof_in_ov=pos,
            pou=pou,
            diameter=_diameter(mesh.vertices[verts]),
            n_triangles=nt,
        )

    coarse = [make(win, m, s, mu_c) for (win, m), s in zip(raw_coarse, coarse_sets)]
    fine = []
    cover = np.zeros(nt, dtype=np.int64)
    for (win, _), fam, fsets in zip(raw_coarse, raw_fine, fine_sets):
        subs = []
        for m, s in zip(fam, fsets):
            subs.append(make(win, m, s, mu_f))
            cover[win.gtri[m]] += 1
        fine.append(subs)
    if cover.min() < 1:
        raise ConfigError("fine subdomains do not cover the mesh")
    return TwoLevelDecomposition(
        coarse=coarse,
        fine=fine,
        coarse_multiplicity=mu_c,
        fine_multiplicity=mu_f,
        Lambda=int(cover.max()),
        Hc=max(s.diameter for s in coarse),
        Hf=max(s.diameter for fam in fine for s in fam),
        layers_c=int(layers_c),
        layers_f=int(layers_f),
    )
