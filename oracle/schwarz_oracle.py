"""CPU oracle of the two-level additive Schwarz apply (TEST INFRASTRUCTURE ONLY).

Restates pkg/src/helmdd/schwarz.py:
  * factorisation of every fine block B[idof][:, idof] with SuperLU defaults
    (schwarz.py:104-110) and lu_factor(B0) (schwarz.py:88-90);
  * apply (schwarz.py:51-61): out = 0; out += Z lu_solve(B0, Z^T r) when a
    coarse space exists; then, subdomain by subdomain in (i, j) order,
    out[idof] += B_s^{-1} r[idof];
  * apply_T (63-65) and apply_coarse (67-71).
"""

import numpy as np
import scipy.linalg
import scipy.sparse as sp
import scipy.sparse.linalg as spla


class OraclePreconditioner:
    def __init__(self, forms, dec, coarse=None, b0_lu=None):
        self.B = sp.csr_matrix(forms.helmholtz)
        self.n = self.B.shape[0]
        Bc = self.B.tocsc()
        self.blocks = []
        for _i, _j, sub in dec.fine_flat():
            idof = np.asarray(sub.idof)
            if idof.size == 0:
                continue
            self.blocks.append((idof, spla.splu(Bc[idof][:, idof].tocsc())))
        self.Z = None
        self.lu = None
        if coarse is not None and coarse.m_total > 0:
            self.Z = sp.csc_matrix(coarse.Z)
            # b0_lu: an existing lu_factor(B0) (identical call) to skip recomputing it
            self.lu = b0_lu if b0_lu is not None else scipy.linalg.lu_factor(np.asarray(coarse.B0))

    def apply(self, r):
        r = np.asarray(r, dtype=float)
        out = np.zeros(self.n)
        if self.Z is not None:
            out += self.Z @ scipy.linalg.lu_solve(self.lu, self.Z.T @ r)
        for idof, lu in self.blocks:
            out[idof] += lu.solve(r[idof])
        return out

    def apply_T(self, u):
        return self.apply(self.B @ np.asarray(u, dtype=float))

    def apply_coarse(self, r):
        if self.Z is None:
            return np.zeros(self.n)
        return self.Z @ scipy.linalg.lu_solve(self.lu, self.Z.T @ np.asarray(r, dtype=float))

    def local_sum(self, r):
        """sum_s E_s B_s^{-1} R_s r alone."""
        out = np.zeros(self.n)
        for idof, lu in self.blocks:
            out[idof] += lu.solve(r[idof])
        return out
