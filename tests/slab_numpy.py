"""Test infrastructure: a numpy implementation of the slab backend interface of
paper_2405_19991_b200/slab.py (the operations of include/otm_slab.h) on CPU torch
tensors, so the slab orchestration and the torch.distributed transport can be
exercised with gloo on CPU.  Restates the same reference formulas as
oracle/otm_oracle.py (solver.py:111-200, homogenize.py:103-122) on ghosted slabs;
the agglomerated coarse levels use an exact pinned pseudo-inverse."""

import numpy as np
import torch

from oracle import otm_oracle as O


def _sh(a, dy, dz):
    """a[..., y + dy, z + dz] with periodic y/z."""
    return np.roll(np.roll(a, -dy, axis=-2), -dz, axis=-1)


def _bits(b):
    return b & 1, (b >> 1) & 1, (b >> 2) & 1


def _apply(A, kap, Kt):
    """K A on the interior planes of a ghosted slab (nxl + 2 planes)."""
    nxl = A.shape[0] - 2
    out = np.zeros((nxl,) + A.shape[1:])
    for q in range(2):
        for jj in range(2):
            for kk in range(2):
                ke = _sh(kap[q:q + nxl], jj - 1, kk - 1)
                a = (1 - q) | ((1 - jj) << 1) | ((1 - kk) << 2)
                e = np.zeros_like(out)
                for b in range(8):
                    bx, by, bz = _bits(b)
                    e += Kt[a, b] * _sh(A[q + bx:q + bx + nxl], jj - 1 + by, kk - 1 + bz)
                out += ke * e
    return out


def _interp(c, axis):
    """Linear interpolation to twice the size along a periodic axis (even: copy, odd: mean)."""
    n = c.shape[axis]
    out_shape = list(c.shape)
    out_shape[axis] = 2 * n
    out = np.zeros(out_shape)
    ev = [slice(None)] * c.ndim
    od = [slice(None)] * c.ndim
    ev[axis] = slice(0, 2 * n, 2)
    od[axis] = slice(1, 2 * n, 2)
    out[tuple(ev)] = c
    out[tuple(od)] = 0.5 * (c + np.roll(c, -1, axis=axis))
    return out


def _fw(a, axis):
    """Full weighting to half the size along a periodic axis."""
    s = 0.25 * np.roll(a, 1, axis=axis) + 0.5 * a + 0.25 * np.roll(a, -1, axis=axis)
    sl = [slice(None)] * a.ndim
    sl[axis] = slice(0, a.shape[axis], 2)
    return s[tuple(sl)]


class NumpySlabBackend:
    device = "cpu"
    f32 = torch.float32
    f64 = torch.float64

    def zeros(self, shape, dtype):
        return torch.zeros(shape, dtype=dtype)

    @staticmethod
    def _n(t):
        return t.numpy().astype(np.float64)

    @staticmethod
    def _w(t, val, interior=True):
        v = torch.from_numpy(np.ascontiguousarray(val)).to(t.dtype)
        if interior:
            t.narrow(-3, 1, t.shape[-3] - 2).copy_(v)
        else:
            t.copy_(v)

    def stencil(self, op, dims, scale, kap, a, f, dinv, omega, o1, o2=None, want_dots=False):
        Kt = O.voxel_template(scale)
        K = self._n(kap)
        dots = np.zeros(3)
        outs1, outs2 = [], []
        for c in range(3):
            if op == 0:
                zc = omega * self._n(dinv) * self._n(f)[c]
                res = self._n(f)[c][1:-1] - _apply(zc, K, Kt)
                outs1.append(zc[1:-1])
                outs2.append(res)
            elif op == 1:
                z = self._n(a)[c]
                fv = self._n(f)[c][1:-1]
                zn = z[1:-1] + omega * self._n(dinv)[1:-1] * (fv - _apply(z, K, Kt))
                outs1.append(zn)
                dots[c] = float((fv * zn).sum())
            else:
                p = self._n(a)[c]
                q = _apply(p, K, Kt)
                outs1.append(q)
                dots[c] = float((p[1:-1] * q).sum())
        self._w(o1, np.stack(outs1))
        if o2 is not None:
            self._w(o2, np.stack(outs2))
        return dots if want_dots else None

    def stencil_range(self, op, dims, scale, kap, a, f, dinv, omega, o1, o2, x_lo, x_hi, want_dots=False):
        """otm_slab_stencil_range: the whole-slab stencil on the arrays as they are now,
        of which only the output planes [x_lo, x_hi) are written; dots over those planes."""
        t1 = o1.clone()
        t2 = o2.clone() if o2 is not None else None
        self.stencil(op, dims, scale, kap, a, f, dinv, omega, t1, t2)
        k = x_hi - x_lo
        o1.narrow(-3, x_lo, k).copy_(t1.narrow(-3, x_lo, k))
        if o2 is not None:
            o2.narrow(-3, x_lo, k).copy_(t2.narrow(-3, x_lo, k))
        if not want_dots:
            return None
        out = self._n(o1)[:, x_lo:x_hi]
        other = self._n(f if op == 1 else a)[:, x_lo:x_hi]
        return (other * out).sum(axis=(1, 2, 3))

    # device-scalar protocol of slab.py (here plain numpy arrays)
    @staticmethod
    def scalars(n):
        return np.zeros(n)

    @staticmethod
    def to_host(S):
        return np.asarray(S)

    @staticmethod
    def put(S, i, v):
        v = np.asarray(v, dtype=np.float64).ravel()
        S[i:i + len(v)] = v

    @staticmethod
    def pcg_step(stage, S):
        """include/otm_slab.h otm_slab_pcg_step, restated."""
        for c in range(3):
            if stage == 0:
                S[6 + c] = 0.0 if S[24] != 0 else (S[c] / S[3 + c] if S[3 + c] != 0 else 0.0)
                S[3 + c] = S[c]
            elif stage == 1:
                S[12 + c] = S[c] / S[9 + c] if (S[21 + c] != 0 and S[9 + c] > 0) else 0.0
            else:
                S[25 + c] += S[21 + c]
                if not (S[15 + c] > S[18 + c]):
                    S[21 + c] = 0.0
        if stage == 0:
            S[24] = 0.0

    def stencil_dev(self, op, dims, scale, kap, a, f, dinv, omega, o1, o2=None):
        return self.stencil(op, dims, scale, kap, a, f, dinv, omega, o1, o2, want_dots=True)

    def pupd_dev(self, dims, z, p, beta):
        return self.pupd(dims, z, p, np.asarray(beta))

    def upd_dev(self, dims, d, r, p, q, alpha):
        return self.upd(dims, d, r, p, q, np.asarray(alpha))

    def restrict(self, dims_f, res_f, f_c):
        R = self._n(res_f)                          # (3, nxl+2, ny, nz)
        nxl = dims_f[0]
        x = 0.25 * R[:, 0:nxl - 1:2] + 0.5 * R[:, 1:nxl:2] + 0.25 * R[:, 2:nxl + 1:2]
        self._w(f_c, _fw(_fw(x, 2), 3))

    def prolong(self, dims_f, z_c, z_f):
        Zc = self._n(z_c)                           # (3, ncl+2, nyc, nzc)
        nxl = dims_f[0]
        yz = _interp(_interp(Zc, 2), 3)
        fine = np.zeros((3, nxl) + yz.shape[2:])
        for x in range(1, nxl + 1):
            j0 = (x + 1) >> 1
            fine[:, x - 1] = yz[:, j0] if x & 1 else 0.5 * (yz[:, j0] + yz[:, j0 + 1])
        zf = self._n(z_f)
        zf[:, 1:-1] += fine
        self._w(z_f, zf, interior=False)

    def coarsen(self, dims_f, k_f, k_c):
        K = self._n(k_f)
        nxl = dims_f[0]
        x = 0.5 * (K[1:nxl:2] + K[2:nxl + 1:2])
        y = 0.5 * (x[:, 0::2] + x[:, 1::2])
        z = 0.5 * (y[:, :, 0::2] + y[:, :, 1::2])
        self._w(k_c, z)

    def dinv(self, dims, scale, kap, out):
        Kt = O.voxel_template(scale)
        K = self._n(kap)
        nxl = dims[0]
        s = np.zeros((nxl,) + K.shape[1:])
        for q in range(2):
            for jj in range(2):
                for kk in range(2):
                    s += _sh(K[q:q + nxl], jj - 1, kk - 1)
        self._w(out, 1.0 / (Kt[0, 0] * s))

    def pupd(self, dims, z, p, beta):
        P, Z = self._n(p), self._n(z)
        for c in range(3):
            P[c, 1:-1] = Z[c, 1:-1] + beta[c] * P[c, 1:-1]
        self._w(p, P, interior=False)

    def upd(self, dims, d, r, p, q, alpha):
        D, R, P, Q = self._n(d), self._n(r), self._n(p), self._n(q)
        rr = np.zeros(3)
        for c in range(3):
            D[c, 1:-1] += alpha[c] * P[c, 1:-1]
            R[c, 1:-1] -= alpha[c] * Q[c, 1:-1]
            rr[c] = float((R[c, 1:-1] ** 2).sum())
        self._w(d, D, interior=False)
        self._w(r, R, interior=False)
        return rr

    def _loads(self, scale, K):
        F0 = O.voxel_template(scale) @ O.CORNER_BITS.astype(np.float64)
        nxl = K.shape[0] - 2
        f = np.zeros((3, nxl) + K.shape[1:])
        for a in range(8):
            ax, ay, az = _bits(a)
            ke = _sh(K[1 - ax:1 - ax + nxl], -ay, -az)
            for c in range(3):
                f[c] += F0[a, c] * ke
        return f

    def load_sums(self, dims, scale, kap64):
        f = self._loads(scale, self._n(kap64))
        return f.reshape(3, -1).sum(axis=1)

    def res64(self, dims, scale, kap64, T, fmean, r32):
        K = self._n(kap64)
        Tn = self._n(T)
        Kt = O.voxel_template(scale)
        f = self._loads(scale, K)
        sums = np.zeros(9)
        rs = []
        for c in range(3):
            r = (f[c] - fmean[c]) - _apply(Tn[c], K, Kt)
            rs.append(r)
            sums[c] = float((r * r).sum())
            sums[3 + c] = float((f[c] * f[c]).sum())
            sums[6 + c] = float(Tn[c, 1:-1].sum())
        self._w(r32, np.stack(rs))
        return sums

    def tupd(self, dims, T, d, mean):
        Tn = self._n(T)
        if d is not None:
            Tn[:, 1:-1] += self._n(d)[:, 1:-1]
        for c in range(3):
            Tn[c, 1:-1] -= mean[c]
        self._w(T, Tn, interior=False)

    def tensor_sums(self, dims, scale, T, kap64):
        Tn, K = self._n(T), self._n(kap64)
        nxl = dims[0]
        Kt = O.voxel_template(scale)
        W = []
        for i in range(3):
            W.append(np.stack([O.CORNER_BITS[a, i] - _sh(Tn[i, 1 + _bits(a)[0]:1 + _bits(a)[0] + nxl],
                                                          _bits(a)[1], _bits(a)[2]) for a in range(8)], axis=-1))
        KW = [w @ Kt for w in W]
        ke = K[1:-1]
        return np.array([float((ke * np.einsum("...a,...a->...", W[i], KW[j])).sum()) for i, j in O.PAIRS])

    def filter(self, mode, dims, radius, material, inp, out, kap64=None):
        offs, w = O.filter_taps(radius)
        R = self._n(inp)
        nxl = dims[0]
        acc = np.zeros((nxl,) + R.shape[1:])
        for o, wk in zip(offs, w):
            dx, dy, dz = (-o[0], -o[1], -o[2]) if mode == 1 else o
            acc += wk * _sh(R[1 + dx:1 + dx + nxl], dy, dz)
        self._w(out, acc)
        if mode != 2:
            return None
        k0, kmin, p = material
        self._w(kap64, kmin + acc ** p * (k0 - kmin))
        r = R[1:-1]
        return np.array([r.sum(), (r ** p).sum(), acc.sum()])

    def sensitivity(self, dims, n_total, material, T, rho_f, dG, sens_f):
        k0, kmin, p = material
        Tn = self._n(T)
        nxl = dims[0]
        Kt = O.voxel_template((1.0, 1.0, 1.0))
        W = []
        for i in range(3):
            W.append(np.stack([O.CORNER_BITS[a, i] - _sh(Tn[i, 1 + _bits(a)[0]:1 + _bits(a)[0] + nxl],
                                                          _bits(a)[1], _bits(a)[2]) for a in range(8)], axis=-1))
        KW = [w @ Kt for w in W]
        con = sum(dG[q] * np.einsum("...a,...a->...", W[i], KW[j]) for q, (i, j) in enumerate(O.PAIRS))
        rf = self._n(rho_f)[1:-1]
        self._w(sens_f, p * rf ** (p - 1.0) * (k0 - kmin) * con / n_total)

    @staticmethod
    def _cand(r, s, n_total, oc, lam):
        desc = n_total * (-s)
        lo = np.maximum(r - oc.step_limit, oc.min_density)
        hi = np.minimum(r + oc.step_limit, 1.0)
        if lam == 0.0:
            return np.where(desc > 0, hi, np.where(desc < 0, lo, r))
        return np.minimum(np.maximum(r * np.maximum(desc / lam, 1e-10) ** oc.damp, lo), hi)

    def oc_sums(self, dims, n_total, oc, rho, sens, lams):
        r, s = self._n(rho)[1:-1], self._n(sens)[1:-1]
        return np.array([self._cand(r, s, n_total, oc, lam).sum() for lam in lams])

    def oc_apply(self, dims, n_total, oc, rho, sens, lam, rho_out):
        r, s = self._n(rho)[1:-1], self._n(sens)[1:-1]
        new = self._cand(r, s, n_total, oc, lam)
        changed = float((new != r).sum())
        self._w(rho_out, new)
        return changed

    # agglomerated levels: exact pinned pseudo-inverse G = P Z P at scale 1
    def coarse_hierarchy(self, dims):
        return {"dims": tuple(dims)}

    def coarse_build(self, ctx, kap_full32):
        dims = ctx["dims"]
        K = kap_full32.numpy().astype(np.float64)
        n = int(np.prod(dims))
        Kt = O.voxel_template((1.0, 1.0, 1.0))
        A = np.zeros((n, n))
        for j in range(n):
            e = np.zeros(n)
            e[j] = 1.0
            E = e.reshape(dims)
            Eg = np.concatenate([E[-1:], E, E[:1]])
            Kg = np.concatenate([K[-1:], K, K[:1]])
            A[:, j] = _apply(Eg, Kg, Kt).ravel()
        Z = np.zeros((n, n))
        Z[1:, 1:] = np.linalg.inv(A[1:, 1:])
        P = np.eye(n) - 1.0 / n
        ctx["G"] = P @ Z @ P

    def coarse_vcycle(self, ctx, f_full, z_full):
        F = f_full.numpy().astype(np.float64).reshape(3, -1)
        Z = (ctx["G"] @ F.T).T
        z_full.copy_(torch.from_numpy(Z.reshape(z_full.shape)).to(z_full.dtype))
