"""Block PCG study (CPU, scipy; not product code): does solving the three load cases
as one block Krylov space (O'Leary block CG, 3x3 alpha/beta) cut the batched
iteration count of the warm-started solves?

    python tools/block_study.py gpurun_out/fields_64_c3.npz 150

Solves the three cases on design it+1, warm-started from the solution on design it
(as the design loop does), to a relative residual of 1e-6 per case: case-wise PCG
(the batched solver runs until the slowest case is done) against block PCG.
"""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
from oracle import otm_oracle as O  # noqa: E402
from solver_study import VCycle  # noqa: E402


def pcg(A, M, b, x0, tol=1e-6, maxit=300):
    b = b - b.mean()
    x = x0.copy()
    r = b - A @ x
    r -= r.mean()
    bn = np.linalg.norm(b)
    if np.linalg.norm(r) / bn <= tol:
        return 0, x
    z = M.apply(r)
    p = z.copy()
    rz = r @ z
    for it in range(1, maxit + 1):
        q = A @ p
        a = rz / (p @ q)
        x += a * p
        r -= a * q
        if np.linalg.norm(r) / bn <= tol:
            return it, x
        z = M.apply(r)
        rz2 = r @ z
        p = z + (rz2 / rz) * p
        rz = rz2
    return maxit, x


def block_pcg(A, M, Bm, X0, tol=1e-6, maxit=300):
    Bm = Bm - Bm.mean(axis=0)
    X = X0.copy()
    R = Bm - A @ X
    R -= R.mean(axis=0)
    bn = np.linalg.norm(Bm, axis=0)
    if (np.linalg.norm(R, axis=0) / bn <= tol).all():
        return 0, X
    Z = np.stack([M.apply(R[:, c]) for c in range(3)], axis=1)
    P = Z.copy()
    RZ = R.T @ Z
    for it in range(1, maxit + 1):
        Q = A @ P
        al = np.linalg.solve(P.T @ Q, RZ)
        X += P @ al
        R -= Q @ al
        if (np.linalg.norm(R, axis=0) / bn <= tol).all():
            return it, X
        Z = np.stack([M.apply(R[:, c]) for c in range(3)], axis=1)
        RZ2 = R.T @ Z
        be = np.linalg.solve(RZ, RZ2)
        P = Z + P @ be
        RZ = RZ2
    return maxit, X


def main():
    data = np.load(sys.argv[1])
    it0 = int(sys.argv[2])
    mat = O.Material()
    sols = None
    for it in (it0, it0 + 1, it0 + 2):
        rho = data[f"rho_{it}"].astype(np.float64)
        kap = O.simp(rho, mat)
        h = O.Hierarchy(rho.shape)
        h.build(kap)
        F = np.stack([O.macro_load(h, i).ravel() for i in range(3)], axis=1)
        M = VCycle(kap, "jac")
        A = M.A[0]
        if sols is None:                     # the previous design's solutions (warm start)
            sols = np.stack([pcg(A, M, F[:, c], np.zeros(F.shape[0]), tol=1e-8)[1] for c in range(3)], axis=1)
            continue
        its, xs = zip(*[pcg(A, M, F[:, c], sols[:, c]) for c in range(3)])
        nb, _ = block_pcg(A, M, F, sols)
        print(f"design {it}: case-wise {list(its)} (batched {max(its)}), block {nb}", flush=True)
        sols = np.stack(xs, axis=1)


if __name__ == "__main__":
    main()
