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
SRC = os.path.join(HERE, "dock_oracle.c")


def build(force: bool = False) -> str:
    if force or not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(SRC):
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
                   ("bump_checks", "<i8"), ("bump_checks_r32", "<i8"), ("bump_early_exits", "<i8")])
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
        L.or_grid_score.restype = C.c_int
        L.or_grid_score.argtypes = [vp, vp, C.c_int]
        L.or_rescore.restype = C.c_int64
        L.or_rescore.argtypes = [vp, vp, vp, C.c_int]
        L.or_rot.restype = None
        L.or_rot.argtypes = [C.c_int, C.c_int, vp]
        L.or_fnv1a64.restype = C.c_uint64
        L.or_fnv1a64.argtypes = [C.c_char_p, C.c_size_t]
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


def dock_batch(batch, pocket, table, cfg, seed: int = 0, threads: Optional[int] = None) -> OracleOutput:
    """Sequential dock_ligand per ligand, OpenMP over ligands."""
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
    rc = lib().or_dock_batch(n, _p(ao), _p(xyz), _p(typ), _p(fo), _p(fax), _p(fm), C.cast(idbuf, C.c_void_p),
                             _p(id_off), C.byref(pk.c), C.byref(ccfg), int(threads or os.cpu_count() or 1),
                             _p(res), _p(rr), _p(rt), _p(bx))
    if rc != 0:
        raise RuntimeError(f"oracle failed ({rc})")
    return OracleOutput(res[:n], rr[:n], rt[:nf], bx[:na])


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
