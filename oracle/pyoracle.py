"""Independent pure-Python restatement of the docking pipeline (TEST INFRASTRUCTURE ONLY).

A second, separately written CPU restatement of SPEC.md's docking module (Alg. 1,
PAPER.md:208-252) under the numeric recipe of DESIGN.md §3, with every f32 operation emulated
exactly (numpy float32 scalars for + - * / sqrt, an exact fused multiply-add below).  It exists
to pin the C oracle (oracle/dock_oracle.c): tests/test_oracle_crosscheck.py requires the two
to agree bit for bit on small ligands.  It is slow (pure-Python loops) and only used on small
cases.
"""
from __future__ import annotations

import math
from typing import List, Sequence, Tuple

import numpy as np

f32 = np.float32
OUTSIDE = -100


def fmaf(a, b, c) -> np.float32:
    """Correctly rounded single-precision a*b + c."""
    a, b, c = float(a), float(b), float(c)
    p = a * b                        # exact: 24-bit x 24-bit significands fit in binary64
    s = math.fsum((p, c))            # binary64 rounding of the exact sum
    r = f32(s)
    if float(r) == s:
        return r
    lo, hi = (r, np.nextafter(r, f32(np.inf))) if float(r) < s else (np.nextafter(r, f32(-np.inf)), r)
    mid = (float(lo) + float(hi)) / 2.0
    if s != mid:
        return r                     # no double-rounding hazard
    e = math.fsum((p, c, -s))        # exact residual decides the side of the tie
    if e > 0:
        return hi
    if e < 0:
        return lo
    return r


def trig(deg: int) -> Tuple[np.float32, np.float32]:
    rad = deg * 0.017453292519943295
    return f32(math.cos(rad)), f32(math.sin(rad))


def rot_x(deg):
    c, s = trig(deg % 360)
    return [f32(1), f32(0), f32(0), f32(0), c, -s, f32(0), s, c]


def rot_y(deg):
    c, s = trig(deg % 360)
    return [c, f32(0), s, f32(0), f32(1), f32(0), -s, f32(0), c]


def rot_z(deg):
    c, s = trig(deg % 360)
    return [c, -s, f32(0), s, c, f32(0), f32(0), f32(0), f32(1)]


def mat3_mul(A, B):
    return [fmaf(A[3 * i + 2], B[6 + j], fmaf(A[3 * i + 1], B[3 + j], f32(A[3 * i] * B[j])))
            for i in range(3) for j in range(3)]


def transform(M, t, d):
    return [fmaf(M[3 * k + 2], d[2], fmaf(M[3 * k + 1], d[1], fmaf(M[3 * k], d[0], t[k]))) for k in range(3)]


def mix64(z: int) -> int:
    m = (1 << 64) - 1
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def fnv1a64(s: str) -> int:
    h = 0xCBF29CE484222325
    for ch in s.encode():
        h = ((h ^ ch) * 0x100000001B3) & ((1 << 64) - 1)
    return h


class Pocket:
    def __init__(self, origin, spacing, dims, values, patoms, ptypes, table, bins):
        self.origin = [f32(o) for o in origin]
        self.s = f32(spacing)
        self.dims = [int(d) for d in dims]
        self.values = np.asarray(values, np.int64).reshape(-1)
        self.inv_s = f32(1.0 / float(self.s))
        self.pat = [[f32((float(p[k]) - float(self.origin[k])) / float(self.s)) for k in range(3)] for p in patoms]
        self.ptype = [int(t) for t in ptypes]
        self.nb = len(bins)
        self.ub2 = [f32((float(b[0]) / float(self.s)) ** 2) for b in bins]
        tab = np.asarray(table, np.float32).reshape(16, 16)
        self.w = {}
        for i in range(16):
            for j in range(16):
                for b, (_, mult) in enumerate(bins):
                    prod = f32(tab[i, j] * f32(mult))
                    self.w[(i, j, b)] = int(round_half_even(float(prod) * 16777216.0))
                self.w[(i, j, self.nb)] = 0

    def value(self, u) -> int:
        n = [f32(np.rint(x)) for x in u]
        for k in range(3):
            if not (n[k] >= 0 and n[k] <= self.dims[k] - 1):
                return OUTSIDE
        return int(self.values[int(n[0]) + self.dims[0] * (int(n[1]) + self.dims[1] * int(n[2]))])

    def score(self, U) -> int:
        return sum(self.value(u) for u in U)


def round_half_even(x: float) -> int:
    return int(np.rint(x))


class Ligand:
    def __init__(self, lid: str, xyz, types, axes, masks):
        A = len(types)
        sm = [math.fsum([]) for _ in range(3)]
        acc = [0.0, 0.0, 0.0]
        for i in range(A):
            for k in range(3):
                acc[k] = acc[k] + float(f32(xyz[i][k]))      # sequential f64 sum (P2)
        c0 = [f32(acc[k] / A) for k in range(3)]
        self.d = [[f32(f32(xyz[i][k]) - c0[k]) for k in range(3)] for i in range(A)]
        self.types = [int(t) for t in types]
        self.H = sum(1 for t in self.types if t != 0)
        self.axes = [tuple(a) for a in axes]
        self.masks = [frozenset(m) for m in masks]
        self.idh = fnv1a64(lid)
        self.A = A


def starting_pose(L: Ligand, P: Pocket, r: int, seed: int):
    g = 0x9E3779B97F4A7C15
    base = L.idh ^ ((seed * g) & ((1 << 64) - 1))
    z = [mix64((base + (r * 8 + k + 1) * g) & ((1 << 64) - 1)) for k in range(6)]
    t = []
    for k in range(3):
        U = f32(f32(z[k] >> 40) * f32(5.9604644775390625e-08))
        t.append(f32(f32(P.dims[k] - 1) * f32(f32(0.1) + f32(f32(0.8) * U))))
    R0 = mat3_mul(rot_z((z[5] >> 32) % 360), mat3_mul(rot_y((z[4] >> 32) % 360), rot_x((z[3] >> 32) % 360)))
    return [f32(x * P.inv_s) for x in R0], t


def rigid_coords(L, R0s, t, ax, ay):
    """Pose (ax, ay): u = Ry(ay) (Rx(ax) R0s d) + t, x rotation first (DESIGN.md §3 P6)."""
    Rp = mat3_mul(rot_x(ax), R0s)
    cy, sy = trig(ay)
    out = []
    for d in L.d:
        v = [fmaf(Rp[3 * k + 2], d[2], fmaf(Rp[3 * k + 1], d[1], f32(Rp[3 * k] * d[0]))) for k in range(3)]
        out.append([fmaf(sy, v[2], fmaf(cy, v[0], t[0])), f32(v[1] + t[1]), fmaf(cy, v[2], fmaf(-sy, v[0], t[2]))])
    return out


def align(L, P, R0s, t, step):
    na = 360 // step
    best = None
    for ix in range(na):
        for iy in range(na):
            s = P.score(rigid_coords(L, R0s, t, ix * step, iy * step))
            if best is None or s > best[0]:
                best = (s, ix, iy)
    return best


def torsion(L, f, U, deg, eps):
    ab, ae = L.axes[f]
    a, b = U[ab], U[ae]
    v = [f32(b[k] - a[k]) for k in range(3)]
    ln = f32(np.sqrt(fmaf(v[2], v[2], fmaf(v[1], v[1], f32(v[0] * v[0])))))
    if not (ln >= eps):
        return None
    out = [list(u) for u in U]
    if deg == 0:
        return out
    kx, ky, kz = (f32(x / ln) for x in v)
    c, s = trig(deg)
    C = f32(f32(1) - c)
    Ckx, Cky, Ckz = f32(C * kx), f32(C * ky), f32(C * kz)
    skx, sky, skz = f32(s * kx), f32(s * ky), f32(s * kz)
    R = [fmaf(Ckx, kx, c), fmaf(Ckx, ky, -skz), fmaf(Ckx, kz, sky),
         fmaf(Cky, kx, skz), fmaf(Cky, ky, c), fmaf(Cky, kz, -skx),
         fmaf(Ckz, kx, -sky), fmaf(Ckz, ky, skx), fmaf(Ckz, kz, c)]
    for i in L.masks[f]:
        w = [f32(U[i][k] - a[k]) for k in range(3)]
        out[i] = transform(R, a, w)
    return out


def bump(L, f, U, bd2) -> bool:
    ab, ae = L.axes[f]
    M = L.masks[f]
    for i in sorted(M):
        for j in range(L.A):
            if j in M or j == ab or j == ae:
                continue
            dx, dy, dz = (f32(U[i][k] - U[j][k]) for k in range(3))
            if fmaf(dz, dz, fmaf(dy, dy, f32(dx * dx))) < bd2:
                return True
    return False


def dock_ligand(L: Ligand, P: Pocket, cfg, seed: int = 0):
    """Returns (status, geom, chem_fx, best_restart, (ax, ay) per restart, torsion indices per restart)."""
    s = float(P.s)
    bd2 = f32((float(cfg.bump_distance) / s) ** 2)
    eps = f32(1e-9 / s)
    thr2 = (float(cfg.similarity_rmsd) / s) ** 2
    nt = 360 // cfg.torsion_step_deg
    U_all, geom, valid, aligns, tors = [], [], [], [], []
    for r in range(cfg.restarts_n):
        R0s, t = starting_pose(L, P, r, seed)
        sc, ix, iy = align(L, P, R0s, t, cfg.alignment_step_deg)
        aligns.append((ix, iy, sc))
        U = rigid_coords(L, R0s, t, ix * cfg.alignment_step_deg, iy * cfg.alignment_step_deg)
        nbumped, tr = 0, []
        for f in range(len(L.axes)):
            best = None
            for a in range(nt):
                cand = torsion(L, f, U, a * cfg.torsion_step_deg, eps)
                if cand is None:
                    if nt > 1:
                        return dict(status=2)
                    cand = [list(u) for u in U]
                if bump(L, f, cand, bd2):
                    continue
                sc = P.score(cand)
                if best is None or sc > best[0]:
                    best = (sc, a, cand)
            if best is None:
                nbumped += 1
                tr.append(255)
            else:
                U = best[2]
                tr.append(best[1])
        valid.append(not (len(L.axes) >= 1 and nbumped == len(L.axes)))
        geom.append(P.score(U))
        U_all.append(U)
        tors.append(tr)
    order = sorted([r for r in range(cfg.restarts_n) if valid[r]], key=lambda r: (-geom[r], r))
    if not order:
        return dict(status=1)
    kept = []
    for c in order:
        if len(kept) >= cfg.rescore_top_k:
            break
        ok = True
        for q in kept:
            tot = 0.0
            for i in range(L.A):
                if L.types[i] == 0:
                    continue
                dx, dy, dz = (float(U_all[c][i][k]) - float(U_all[q][i][k]) for k in range(3))
                tt = dx * dx
                tt = tt + dy * dy
                tt = tt + dz * dz
                tot = tot + tt
            ok = ok and (L.H > 0 and tot >= thr2 * L.H)
        if ok:
            kept.append(c)
    best_r, best_c = None, None
    for r in kept:
        acc = 0
        for i in range(L.A):
            for j, pj in enumerate(P.pat):
                dx, dy, dz = (f32(U_all[r][i][k] - pj[k]) for k in range(3))
                d2 = fmaf(dz, dz, fmaf(dy, dy, f32(dx * dx)))
                b = sum(1 for q in range(P.nb) if not (d2 < P.ub2[q]))
                acc += P.w[(L.types[i], P.ptype[j], b)]
        if best_r is None or acc > best_c or (acc == best_c and r < best_r):
            best_r, best_c = r, acc
    return dict(status=0, geom=geom[best_r], chem_fx=best_c, best_restart=best_r, aligns=aligns, tors=tors,
                final_geom=geom, valid=valid, kept=kept)
