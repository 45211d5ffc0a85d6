"""Preconditioner study on dumped designs (CPU, scipy.sparse; not product code).

    python tools/solver_study.py gpurun_out/fields_64_c2.npz [iters...]

For each dumped filtered density: PCG iterations (all three macro loads) to a
relative residual of 1e-6 from zero, and the mean contraction per iteration, for
V-cycle variants:
  jac      damped Jacobi 0.95 / 1.25, 1+1 sweeps, rediscretised child-mean coarse
           operators (libotm's preconditioner)
  jac2     the same with 2+2 sweeps
  cheb2    Chebyshev degree-2 smoother on D^-1 A (eigen bound 1.5), 1+1
  gal      damped Jacobi 1+1 on Galerkin coarse operators R A P
  gal_cheb Chebyshev 1+1 on Galerkin operators
Uses the oracle's operator assembly (test infrastructure) for the fine matrix.
"""
import sys

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, ".")
from oracle import otm_oracle as O  # noqa: E402


def level_matrix(lev):
    dims = lev.dims
    n = int(np.prod(dims))
    idx = np.arange(n).reshape(dims)
    rows, cols, vals = [], [], []
    for d, W in lev.coef.items():
        rows.append(idx.ravel())
        cols.append(O._shifted(idx, d).ravel())
        vals.append(W.ravel())
    return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n))


def prolongation(fine, coarse):
    """Trilinear periodic interpolation coarse -> fine as a sparse matrix (solver.py:180-200)."""
    mats = []
    for ax in range(3):
        nf, nc = fine[ax], coarse[ax]
        if nc == nf:
            mats.append(sp.identity(nf, format="csr"))
            continue
        r, c, v = [], [], []
        for i in range(nc):
            r += [2 * i, 2 * i + 1, 2 * i + 1]
            c += [i, i, (i + 1) % nc]
            v += [1.0, 0.5, 0.5]
        mats.append(sp.csr_matrix((v, (r, c)), shape=(nf, nc)))
    return sp.kron(sp.kron(mats[0], mats[1]), mats[2]).tocsr()


class VCycle:
    def __init__(self, kappa, variant):
        self.variant = variant
        chain = O.level_chain(kappa.shape)
        h = O.Hierarchy(kappa.shape)
        h.build(kappa)
        self.A = [level_matrix(h.levels[0])]
        self.P = []
        for li in range(1, len(chain)):
            P = prolongation(chain[li - 1][0], chain[li][0])
            self.P.append(P)
            if variant.startswith("gal"):
                self.A.append((P.T @ self.A[-1] @ P / 8.0).tocsr())
            else:
                self.A.append(level_matrix(h.levels[li]))
        self.Dinv = [1.0 / A.diagonal() for A in self.A]
        Ac = self.A[-1].toarray()
        red = Ac[1:, 1:]
        self.Ginv = np.linalg.inv(red)
        self.sweeps = 2 if variant == "jac2" else 1

    def smooth(self, l, x, b, zero):
        A, Di = self.A[l], self.Dinv[l]
        if "cheb" in self.variant:
            # Chebyshev degree 2 on [lmax/4, lmax], lmax = 1.5 (Rayleigh bound)
            lmax, lmin = 1.5, 1.5 / 4.0
            th, de = (lmax + lmin) / 2, (lmax - lmin) / 2
            r = b - (A @ x if not zero else 0.0)
            d = Di * r / th
            x = x + d
            rho_old = de / th
            sig = th / de
            for _ in range(1):
                r = b - A @ x
                rho = 1.0 / (2 * sig - rho_old)
                d = rho * rho_old * d + 2 * rho / de * Di * r
                x = x + d
                rho_old = rho
            return x
        w = 0.95 if l == 0 else 1.25
        for s in range(self.sweeps):
            if zero and s == 0:
                x = w * Di * b
            else:
                x = x + w * Di * (b - A @ x)
        return x

    def apply(self, b, l=0):
        if l == len(self.A) - 1:
            f = b - b.mean()
            x = np.zeros_like(f)
            x[1:] = self.Ginv @ f[1:]
            return x - x.mean()
        x = self.smooth(l, np.zeros_like(b), b, True)
        r = b - self.A[l] @ x
        bc = self.P[l].T @ r / 8.0
        xc = self.apply(bc, l + 1)
        x = x + self.P[l] @ xc
        return self.smooth(l, x, b, False)


def pcg(A, M, b, tol=1e-6, maxit=300):
    b = b - b.mean()
    x = np.zeros_like(b)
    r = b.copy()
    z = M.apply(r)
    p = z.copy()
    rz = r @ z
    bn = np.linalg.norm(b)
    hist = [1.0]
    for it in range(1, maxit + 1):
        q = A @ p
        a = rz / (p @ q)
        x += a * p
        r -= a * q
        hist.append(np.linalg.norm(r) / bn)
        if hist[-1] <= tol:
            return it, hist
        z = M.apply(r)
        rz2 = r @ z
        p = z + (rz2 / rz) * p
        rz = rz2
    return maxit, hist


def main():
    data = np.load(sys.argv[1])
    keys = sorted((k for k in data if k.startswith("rho_")), key=lambda k: int(k[4:]))
    want = set(sys.argv[2:])
    variants = ["jac", "jac2", "cheb2", "gal", "gal_cheb"]
    mat = O.Material()
    for k in keys:
        if want and k[4:] not in want:
            continue
        rho = data[k].astype(np.float64)
        kap = O.simp(rho, mat)
        h = O.Hierarchy(rho.shape)
        h.build(kap)
        loads = [O.macro_load(h, i).ravel() for i in range(3)]
        line = [f"{k}:"]
        for v in variants:
            M = VCycle(kap, v)
            its = []
            for f in loads:
                it, hist = pcg(M.A[0], M, f)
                its.append(it)
            rate = np.exp(np.log(1e-6) / np.mean(its))
            line.append(f"{v} {its} ({rate:.3f})")
        print("  ".join(line), flush=True)


if __name__ == "__main__":
    main()
