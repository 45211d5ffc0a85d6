"""Krylov recycling study (CPU, scipy; not product code): does projecting the warm
start onto the previous solve's search directions cut PCG iterations?

    python tools/recycle_study.py gpurun_out/fields_64_c3.npz 150

Solves case 0 on designs it-1, it, it+1 in sequence (warm starts), keeping the
search directions P and K P of the solve on design `it`; the solve on it+1 then
starts from x0 = x_warm + sum_i p_i (p_i . r0) / (p_i . K_old p_i) (the old K's
conjugacy, no new operator applications) -- iterations to 1e-6 with and without.
"""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
from oracle import otm_oracle as O  # noqa: E402
from solver_study import VCycle  # noqa: E402


def pcg(A, M, b, x0, tol=1e-6, maxit=300, keep=False):
    b = b - b.mean()
    x = x0.copy()
    r = b - A @ x
    r -= r.mean()
    z = M.apply(r)
    p = z.copy()
    rz = r @ z
    bn = np.linalg.norm(b)
    P, Q = [], []
    if np.linalg.norm(r) / bn <= tol:
        return 0, x, P, Q
    for it in range(1, maxit + 1):
        q = A @ p
        pq = p @ q
        a = rz / pq
        if keep:
            P.append(p.copy())
            Q.append(pq)
        x += a * p
        r -= a * q
        if np.linalg.norm(r) / bn <= tol:
            return it, x, P, Q
        z = M.apply(r)
        rz2 = r @ z
        p = z + (rz2 / rz) * p
        rz = rz2
    return maxit, x, P, Q


def main():
    data = np.load(sys.argv[1])
    it0 = int(sys.argv[2])
    mat = O.Material()
    x = None
    P = Q = None
    for k, it in enumerate((it0, it0 + 1, it0 + 2)):
        rho = data[f"rho_{it}"].astype(np.float64)
        kap = O.simp(rho, mat)
        h = O.Hierarchy(rho.shape)
        h.build(kap)
        f = O.macro_load(h, 0).ravel()
        M = VCycle(kap, "jac")
        A = M.A[0]
        x0 = np.zeros_like(f) if x is None else x
        n_plain, xp, P1, Q1 = pcg(A, M, f, x0, keep=True)
        line = f"design {it}: warm {n_plain} iterations"
        if P is not None:
            r0 = (f - f.mean()) - A @ x0
            xr = x0.copy()
            for p, pq in zip(P, Q):
                xr += p * ((p @ r0) / pq)
            n_rec, _, _, _ = pcg(A, M, f, xr)
            line += f"; recycled start ({len(P)} directions): {n_rec} iterations"
        print(line, flush=True)
        x, P, Q = xp, P1, Q1


if __name__ == "__main__":
    main()
