"""ctypes wrapper of the CPU ORACLE (oracle/dock_oracle.c) — test infrastructure only.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import this module; the
product package never does.  See dock_oracle.c's header for what it restates and how it is
pinned.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "liboracle.so")
SRCS = [os.path.join(HERE, f) for f in ("dock_oracle.c", "gen_oracle.c", "Makefile")]


def build(force: bool = False) -> str:
    if force or not os.path.exists(SO) or any(os.path.getmtime(SO) < os.path.getmtime(f) for f in SRCS):
        subprocess.check_call(["make", "-s", "-C", HERE])
    return SO


class OrPocket(C.Structure):
    _fields_ = [("origin", C.c_float * 3), ("spacing", C.c_float), ("dims", C.c_int32 * 3), ("values", C.c_void_p),
                ("n_atoms", C.c_int32), ("atom_xyz", C.c_void_p), ("atom_type", C.c_void_p), ("table", C.c_void_p),
                ("n_bins", C.c_int32), ("bin_ub", C.c_void_p), ("bin_mult", C.c_void_p)]


class OrConfig(C.Structure):
    _fields_ = [("restarts_n", C.c_int32), ("rescore_top_k", C.c_int32), ("alignment_step_deg", C.c_int32),
                ("torsion_step_deg", C.c_int32), ("bump_distance", C.c_float), ("similarity_rmsd", C.c_float),
                ("rescore_cutoff", C.c_float), ("early_exit", C.c_int32), ("seed", C.c_int64)]


RESULT = np.dtype([("status", "<i4"), ("geom_score", "<i4"), ("chem_fx", "<i8"), ("best_restart", "<i4"),
                   ("best_ax", "<i4"), ("best_ay", "<i4"), ("n_kept", "<i4"), ("poses_scored", "<i8"),
                   ("bump_checks", "<i8"), ("bump_checks_rows", "<i8"), ("bump_early_exits", "<i8")])
RESTART = np.dtype([("align_score", "<i4"), ("final_geom", "<i4"), ("ax", "<i4"), ("ay", "<i4"), ("valid", "<i4"),
                    ("kept", "<i4")])

_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        vp = C.c_void_p
        L.or_dock_batch.restype = C.c_int
        L.or_dock_batch.argtypes = [C.c_int] + [vp] * 10 + [C.c_int, vp, vp, vp, vp]
        L.or_dock_batch_latency.restype = C.c_int
        L.or_dock_batch_latency.argtypes = [C.c_int] + [vp] * 10 + [C.c_int, vp, vp, vp, vp]
        L.or_grid_score.restype = C.c_int
        L.or_grid_score.argtypes = [vp, vp, C.c_int]
        L.or_rescore.restype = C.c_int64
        L.or_rescore.argtypes = [vp, vp, vp, C.c_int]
        L.or_rot.restype = None
        L.or_rot.argtypes = [C.c_int, C.c_int, vp]
        L.or_fnv1a64.restype = C.c_uint64
        L.or_fnv1a64.argtypes = [C.c_char_p, C.c_size_t]
        L.or_dock_batch_poses.restype = C.c_int
        L.or_dock_batch_poses.argtypes = [C.c_int] + [vp] * 10 + [C.c_int, vp, vp, vp, vp, vp]
        for name, args in (("or_apply_rigid", [C.c_int, C.c_int, vp, vp, vp, vp]),
                           ("or_apply_torsion", [C.c_int, C.c_int, vp, C.c_int, C.c_int, vp, C.c_int, vp, vp]),
                           ("or_bump_check", [C.c_int, C.c_int, vp, C.c_int, C.c_int, vp, C.c_float, C.c_int, vp,
                                              vp])):
            fn = getattr(L, name)
            fn.restype = None
            fn.argtypes = args
        i32, i64 = C.c_int32, C.c_int64
        for name, args in (("go_generated_id", [i64, i64, C.c_char_p, C.c_size_t]),
                           ("go_mixed_shapes", [i64, i64, i32, i32, i32, i32, vp]),
                           ("go_generate_ligands", [i64, i64, i32] + [vp] * 7),
                           ("go_pocket_atoms", [i64, i32, C.c_float, C.c_float, vp, vp]),
                           ("go_build_pocket", [vp, i32, C.c_float, C.c_float, vp, vp, vp]),
                           ("go_default_table", [i64, vp])):
            fn = getattr(L, name)
            fn.restype = C.c_int
            fn.argtypes = args
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


class _PocketC:
    def __init__(self, pocket, table):
        xyz, typ = pocket.atom_arrays()
        self.keep = [np.ascontiguousarray(pocket.grid_values, dtype=np.int32), np.ascontiguousarray(xyz, np.float32),
                     np.ascontiguousarray(typ, np.uint8) if len(typ) else np.zeros(1, np.uint8),
                     np.ascontiguousarray(table.table, np.float32).reshape(-1),
                     np.array([b[0] for b in table.bins], np.float32), np.array([b[1] for b in table.bins], np.float32)]
        if self.keep[1].size == 0:
            self.keep[1] = np.zeros((1, 3), np.float32)
        p = OrPocket()
        for k in range(3):
            p.origin[k] = pocket.grid_origin[k]
            p.dims[k] = pocket.grid_dims[k]
        p.spacing = pocket.grid_spacing
        p.values = _p(self.keep[0])
        p.n_atoms = len(pocket.pocket_atoms)
        p.atom_xyz, p.atom_type, p.table = _p(self.keep[1]), _p(self.keep[2]), _p(self.keep[3])
        p.n_bins = len(table.bins)
        p.bin_ub, p.bin_mult = _p(self.keep[4]), _p(self.keep[5])
        self.c = p


def _cfg(cfg, seed):
    c = OrConfig()
    c.restarts_n, c.rescore_top_k = cfg.restarts_n, cfg.rescore_top_k
    c.alignment_step_deg, c.torsion_step_deg = cfg.alignment_step_deg, cfg.torsion_step_deg
    c.bump_distance, c.similarity_rmsd, c.rescore_cutoff = cfg.bump_distance, cfg.similarity_rmsd, cfg.rescore_cutoff
    c.early_exit = 1 if cfg.early_exit else 0
    c.seed = seed
    return c


@dataclass
class OracleOutput:
    results: np.ndarray
    restarts: np.ndarray
    restart_torsion: np.ndarray
    best_coords: np.ndarray


def dock_batch(batch, pocket, table, cfg, seed: int = 0, threads: Optional[int] = None,
               latency: bool = False, restart_poses: bool = False) -> OracleOutput:
    """Sequential dock_ligand per ligand, OpenMP over ligands (the batched engine's CPU
    shape); latency=True: ligands one after another, each ligand's restarts on an inner pool of
    `threads` workers (the latency engine's CPU shape) — identical results."""
    n, N = batch.n, cfg.restarts_n
    ids, id_off = batch.id_bytes()
    idbuf = C.create_string_buffer(ids, max(len(ids), 1))
    pk = _PocketC(pocket, table)
    ccfg = _cfg(cfg, seed)
    res = np.zeros(max(n, 1), RESULT)
    rr = np.zeros((max(n, 1), N), RESTART)
    nf, na = int(batch.frag_off[-1]), int(batch.atom_off[-1])
    rt = np.zeros((max(nf, 1), N), np.uint8)
    bx = np.zeros((max(na, 1), 3), np.float32)
    c = np.ascontiguousarray
    ao, xyz, typ = c(batch.atom_off, np.int32), c(batch.atom_xyz, np.float32), c(batch.atom_type, np.uint8)
    fo, fax, fm = c(batch.frag_off, np.int32), c(batch.frag_axis, np.int32), c(batch.frag_mask, np.uint32)
    if fax.size == 0:
        fax, fm = np.zeros((1, 2), np.int32), np.zeros((1, 5), np.uint32)
    args = [n, _p(ao), _p(xyz), _p(typ), _p(fo), _p(fax), _p(fm), C.cast(idbuf, C.c_void_p), _p(id_off),
            C.byref(pk.c), C.byref(ccfg), int(threads or os.cpu_count() or 1), _p(res), _p(rr), _p(rt), _p(bx)]
    rx = None
    if restart_poses:
        rx = np.zeros((max(na, 1) * N, 3), np.float32)
        rc = lib().or_dock_batch_poses(*args, _p(rx))
    else:
        rc = (lib().or_dock_batch_latency if latency else lib().or_dock_batch)(*args)
    if rc != 0:
        raise RuntimeError(f"oracle failed ({rc})")
    out = OracleOutput(res[:n], rr[:n], rt[:nf], bx[:na])
    out.restart_xyz = rx   # [(atom_off[i] * N + r * A_i + a)] rows, Å
    return out


def grid_score(pocket, table, coords) -> int:
    pk = _PocketC(pocket, table)
    x = np.ascontiguousarray(coords, np.float32).reshape(-1, 3)
    return int(lib().or_grid_score(C.byref(pk.c), _p(x), len(x)))


def rescore_fx(pocket, table, coords, types) -> int:
    pk = _PocketC(pocket, table)
    x = np.ascontiguousarray(coords, np.float32).reshape(-1, 3)
    t = np.ascontiguousarray(types, np.uint8)
    return int(lib().or_rescore(C.byref(pk.c), _p(x), _p(t), len(x)))


def rot(axis: int, deg: int) -> np.ndarray:
    m = np.zeros(9, np.float32)
    lib().or_rot(axis, deg, _p(m))
    return m.reshape(3, 3)


def fnv1a64(s: str) -> int:
    b = s.encode()
    return int(lib().or_fnv1a64(b, len(b)))


# ---- oracle-side input makers (gen_oracle.c): the reference arm of bench.py builds its inputs with
# these so its process never loads the product library ------------------------------------------
class OracleBatch:
    """The packed CSR ligand arrays dock_batch consumes (same field names as the product's LigandBatch)."""

    def __init__(self, atom_off, atom_xyz, atom_type, frag_off, frag_axis, frag_mask, ids):
        self.atom_off, self.atom_xyz, self.atom_type = atom_off, atom_xyz, atom_type
        self.frag_off, self.frag_axis, self.frag_mask, self.ids = frag_off, frag_axis, frag_mask, ids

    @property
    def n(self) -> int:
        return len(self.atom_off) - 1

    def id_bytes(self):
        raw = [s.encode() for s in self.ids]
        off = np.zeros(len(raw) + 1, np.int64)
        off[1:] = np.cumsum([len(b) for b in raw]) if raw else []
        return b"".join(raw), off


def generated_id(seed: int, index: int) -> str:
    buf = C.create_string_buffer(64)
    n = lib().go_generated_id(int(seed), int(index), buf, 64)
    return buf.raw[:n].decode()


def mixed_shapes(count: int, seed: int, first_index: int = 0, heavy_range=(8, 40), frag_max: int = 20) -> np.ndarray:
    out = np.zeros((count, 2), np.int32)
    if lib().go_mixed_shapes(int(seed), int(first_index), int(count), int(heavy_range[0]), int(heavy_range[1]),
                             int(frag_max), _p(out)) != 0:
        raise ValueError("bad mixed-shape arguments")
    return out


def generate_batch(shapes: np.ndarray, seed: int, first_index: int = 0) -> OracleBatch:
    """SPEC.md:443 generate_dataset (oracle restatement) for ligands first_index + i of these shapes."""
    shapes = np.ascontiguousarray(np.asarray(shapes, np.int32).reshape(-1, 2))
    n = len(shapes)
    ao, fo = np.zeros(n + 1, np.int32), np.zeros(n + 1, np.int32)
    L = lib()
    if L.go_generate_ligands(int(seed), int(first_index), n, _p(shapes), _p(ao), _p(fo), None, None, None, None):
        raise ValueError("InfeasibleShape")
    na, nf = int(ao[-1]), int(fo[-1])
    xyz, typ = np.zeros((max(na, 1), 3), np.float32), np.zeros(max(na, 1), np.uint8)
    axis, mask = np.zeros((max(nf, 1), 2), np.int32), np.zeros((max(nf, 1), 5), np.uint32)
    L.go_generate_ligands(int(seed), int(first_index), n, _p(shapes), _p(ao), _p(fo), _p(xyz), _p(typ), _p(axis),
                          _p(mask))
    ids = [generated_id(seed, first_index + i) for i in range(n)]
    return OracleBatch(ao, xyz[:na], typ[:na], fo, axis[:nf], mask[:nf], ids)


def generate_mixed_batch(count: int, seed: int, first_index: int = 0, heavy_range=(8, 40),
                         frag_max: int = 20) -> OracleBatch:
    return generate_batch(mixed_shapes(count, seed, first_index, heavy_range, frag_max), seed, first_index)


class OracleTable:
    """InteractionTable as the oracle reads it: .table (16x16) and .bins."""

    def __init__(self, table, bins=((2.0, 0.5), (4.0, 1.0), (6.0, 0.5), (8.0, 0.25))):
        self.table, self.bins = table, tuple(bins)


def default_table(seed: int = 11) -> OracleTable:
    t = np.zeros(256, np.float32)
    lib().go_default_table(int(seed), _p(t))
    return OracleTable(t.reshape(16, 16))


def synthetic_pocket(spacing: float = 0.5, n_atoms: int = 200, seed: int = 7, rmin: float = 7.0, rmax: float = 10.0,
                     padding: float = 4.0):
    """The shared synthetic pocket built by the oracle restatement of build_pocket; a
    plain model.Pocket (pure Python, no product library)."""
    from paper_2209_05069_b200 import model
    xyz, typ = np.zeros((n_atoms, 3), np.float32), np.zeros(n_atoms, np.uint8)
    L = lib()
    L.go_pocket_atoms(int(seed), int(n_atoms), float(rmin), float(rmax), _p(xyz), _p(typ))
    origin, dims = (C.c_float * 3)(), (C.c_int32 * 3)()
    if L.go_build_pocket(_p(xyz), n_atoms, float(spacing), float(padding), origin, dims, None):
        raise ValueError("EmptyPocket")
    vals = np.zeros(int(dims[0]) * int(dims[1]) * int(dims[2]), np.int32)
    L.go_build_pocket(_p(xyz), n_atoms, float(spacing), float(padding), origin, dims, _p(vals))
    atoms = tuple(model.Atom.of(*xyz[i], int(typ[i])) for i in range(n_atoms))
    return model.Pocket(tuple(float(o) for o in origin), float(np.float32(spacing)), tuple(int(d) for d in dims), vals,
                        atoms)


# ---- the other L2 ops in Å, batched over poses [P, n, 3] ----------------------
def _mask_words(mask) -> np.ndarray:
    m = np.zeros(5, np.uint32)
    for i in mask:
        m[int(i) >> 5] |= np.uint32(1 << (int(i) & 31))
    return m


def apply_rigid(coords, m, center) -> np.ndarray:
    P = np.ascontiguousarray(coords, np.float32).reshape(-1, np.shape(coords)[-2], 3)
    mm = np.ascontiguousarray(np.broadcast_to(np.asarray(m, np.float32).reshape(-1, 9), (P.shape[0], 9)))
    cc = np.ascontiguousarray(np.broadcast_to(np.asarray(center, np.float32).reshape(-1, 3), (P.shape[0], 3)))
    out = np.empty_like(P)
    lib().or_apply_rigid(P.shape[1], P.shape[0], _p(P), _p(mm), _p(cc), _p(out))
    return out


def apply_torsion(coords, axis_begin: int, axis_end: int, mask, deg: int):
    P = np.ascontiguousarray(coords, np.float32).reshape(-1, np.shape(coords)[-2], 3)
    out = np.empty_like(P)
    st = np.zeros(P.shape[0], np.int32)
    lib().or_apply_torsion(P.shape[1], P.shape[0], _p(P), int(axis_begin), int(axis_end), _p(_mask_words(mask)),
                           int(deg), _p(out), _p(st))
    return out, st


def bump_check(coords, axis_begin: int, axis_end: int, mask, bump_distance: float, early_exit: bool):
    P = np.ascontiguousarray(coords, np.float32).reshape(-1, np.shape(coords)[-2], 3)
    bump = np.zeros(P.shape[0], np.uint8)
    pairs = np.zeros(P.shape[0], np.int64)
    lib().or_bump_check(P.shape[1], P.shape[0], _p(P), int(axis_begin), int(axis_end), _p(_mask_words(mask)),
                        float(bump_distance), int(bool(early_exit)), _p(bump), _p(pairs))
    return bump.astype(bool), pairs
