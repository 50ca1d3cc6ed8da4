"""ctypes binding of libdockscreen.so (include/dockscreen.h) and the packed batch layout.

This is the B200 occupant of the reference's native slot `dockscreen.kernels._core`
(pkg/setup.py:10-18).  The reference falls back to NumPy when its extension is missing
(pkg/setup.py:21-22); this package has NO fallback: `lib()` raises NativeUnavailable when the
shared library is absent, and every docking call raises when no CUDA device is visible.
ctypes releases the GIL for the duration of each call, so engine threads overlap.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
import weakref
from dataclasses import dataclass
from typing import Tuple, List, Optional, Sequence
import collections.abc as _abc

import numpy as np

from . import model

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DOCKSCREEN_LIB") or os.path.join(_HERE, "libdockscreen.so")  # override: A/B builds


def source_sha16() -> str:
    """sha256[:16] over the CUDA sources and build recipe of libdockscreen.so (csrc/*.cu, *.cuh — the
    kernels and their launch code — and the Makefile's flags; not the host-only helpers in
    ds_host.cpp): the identity of the kernels a build contains.  nvcc's output is not
    byte-reproducible (host object paths / temporaries), so profiles are tied to builds by this,
    not by the .so bytes."""
    import hashlib
    h = hashlib.sha256()
    csrc = os.path.join(_HERE, "csrc")
    files = sorted(f for f in os.listdir(csrc) if f.endswith((".cu", ".cuh")) or f == "Makefile")
    for f in files:
        h.update(f.encode())
        with open(os.path.join(csrc, f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]

DS_OK = 0
ERRORS = {
    -1: ValueError, -2: model.TooManyAtoms, -3: model.MalformedFragment, -4: model.IndexOutOfRange,
    -5: model.DegenerateAxis, -6: model.EmptyPocket, -7: model.InfeasibleShape,
}
STATUS_OK, STATUS_NO_VALID_POSE, STATUS_DEGENERATE_AXIS = 0, 1, 2
FAMILY_BATCHED, FAMILY_LATENCY = 0, 1
MASK_WORDS, FRAG_WORDS, MAX_RESTARTS, TORSION_NONE = 5, 8, 32, 255
MAX_BINS = 8
CHEM_SCALE = float(1 << 24)


class NativeUnavailable(RuntimeError):
    """libdockscreen.so is missing or a CUDA device is not usable — no fallback exists."""


class DsError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"libdockscreen error {code}: {msg}")
        self.code = code


# ---- ABI structs (mirror include/dockscreen.h) -----------------------------------------
class PocketDesc(C.Structure):
    _fields_ = [("origin", C.c_float * 3), ("spacing", C.c_float), ("dims", C.c_int32 * 3),
                ("n_atoms", C.c_int32), ("values", C.c_void_p), ("atom_xyz", C.c_void_p),
                ("atom_type", C.c_void_p), ("table", C.c_void_p), ("n_bins", C.c_int32),
                ("bin_ub", C.c_void_p), ("bin_mult", C.c_void_p)]


class DockConfigC(C.Structure):
    _fields_ = [("restarts_n", C.c_int32), ("rescore_top_k", C.c_int32), ("alignment_step_deg", C.c_int32),
                ("torsion_step_deg", C.c_int32), ("bump_distance", C.c_float), ("similarity_rmsd", C.c_float),
                ("rescore_cutoff", C.c_float), ("early_exit", C.c_int32), ("seed", C.c_int64)]


class BatchDesc(C.Structure):
    _fields_ = [("n_ligands", C.c_int32), ("reserved", C.c_int32), ("atom_off", C.c_void_p),
                ("atom_xyzt", C.c_void_p), ("frag_off", C.c_void_p), ("frag_desc", C.c_void_p),
                ("id_hash", C.c_void_p)]


class Outputs(C.Structure):
    _fields_ = [("results", C.c_void_p), ("best_coords", C.c_void_p), ("best_torsion", C.c_void_p),
                ("restarts", C.c_void_p), ("restart_torsion", C.c_void_p)]


class Stats(C.Structure):
    _fields_ = [("total_ms", C.c_float), ("align_ms", C.c_float), ("optimize_ms", C.c_float),
                ("launches", C.c_int32), ("select_ms", C.c_float), ("h2d_bytes", C.c_int64),
                ("d2h_bytes", C.c_int64), ("lat_spread", C.c_int32)]


RESULT_DTYPE = np.dtype([("status", "<i4"), ("geom_score", "<i4"), ("chem_fx", "<i8"), ("best_restart", "u1"),
                         ("best_ax", "u1"), ("best_ay", "u1"), ("n_kept", "u1"), ("poses_scored", "<u4"),
                         ("bump_checks", "<u4"), ("bump_early_exits", "<u4")])
RESTART_DTYPE = np.dtype([("align_score", "<i4"), ("final_geom", "<i4"), ("ax", "u1"), ("ay", "u1"),
                          ("valid", "u1"), ("kept", "u1"), ("reserved", "<i4")])
assert RESULT_DTYPE.itemsize == 32 and RESTART_DTYPE.itemsize == 16

_lib = None
_lib_lock = threading.Lock()


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


def lib():
    """Load libdockscreen.so (fails loudly; there is no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailable(f"{LIB_PATH} not built (run __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64, u64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64
        sig = {
            "ds_abi_version": (C.c_int, []), "ds_last_error": (C.c_char_p, []),
            "ds_device_count": (C.c_int, [vp]), "ds_create": (C.c_int, [C.c_int, vp]),
            "ds_destroy": (None, [vp]), "ds_ctx_alloc_count": (C.c_int, [vp, vp]),
            "ds_ctx_stream": (vp, [vp]), "ds_synchronize": (C.c_int, [vp]),
            "ds_host_alloc": (vp, [C.c_size_t]), "ds_host_free": (None, [vp]),
            "ds_ctx_reserve": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, vp]),
            "ds_pocket_create": (C.c_int, [vp, vp, vp]), "ds_pocket_destroy": (None, [vp]),
            "ds_dock": (C.c_int, [vp, vp, vp, vp, C.c_int, vp, vp]),
            "ds_batch_upload": (C.c_int, [vp, vp, vp]),
            "ds_dock_resident": (C.c_int, [vp, vp, vp, vp, C.c_int, vp]),
            "ds_batch_download": (C.c_int, [vp, vp, vp]), "ds_batch_destroy": (None, [vp]),
            "ds_query_capacity": (C.c_int, [vp, C.c_int, vp]),
            "ds_op_grid_score": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, vp]),
            "ds_op_rescore": (C.c_int, [vp, vp, vp, vp, C.c_int, C.c_int, C.c_float, vp]),
            "ds_ligand_id_hash": (u64, [C.c_char_p, C.c_size_t]),
            "ds_generated_id": (C.c_int, [i64, i64, C.c_char_p, C.c_size_t]),
            "ds_generated_ids": (C.c_int, [i64, i64, i32, C.c_void_p, C.c_void_p]),
            "ds_mixed_shapes": (C.c_int, [i64, i64, i32, i32, i32, i32, vp]),
            "ds_generate_ligands": (C.c_int, [i64, i64, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
            "ds_pack_ligands": (C.c_int, [i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
            "ds_generate_pocket_atoms": (C.c_int, [i64, i32, C.c_float, C.c_float, vp, vp]),
            "ds_build_pocket_grid": (C.c_int, [vp, i32, C.c_float, C.c_float, vp, vp, vp]),
            "ds_build_pocket_grid_device": (C.c_int, [vp, vp, i32, C.c_float, C.c_float, vp, vp, vp, vp]),
            "ds_default_table": (C.c_int, [i64, vp]),
            "ds_ligq_parse": (C.c_int, [C.c_char_p, i64, i32, vp, vp, C.c_char_p, i32]),
            "ds_ligq_fill": (C.c_int, [vp] * 11),
            "ds_ligq_free": (None, [vp]),
            "ds_validate_ligands": (C.c_int, [i32] + [vp] * 10),
            "ds_generate_resident": (C.c_int, [vp, i64, i64, i32, vp, vp, vp]),
            "ds_batch_read_inputs": (C.c_int, [vp, vp, vp, vp, vp]),
            "ds_csr_gather": (C.c_int, [i32, vp, vp, vp, i32, vp, vp]),
            "ds_op_apply_rigid": (C.c_int, [vp, vp, i32, i32, vp, vp, vp]),
            "ds_op_apply_torsion": (C.c_int, [vp, vp, i32, i32, i32, i32, vp, i32, vp, vp]),
            "ds_op_bump_check": (C.c_int, [vp, vp, i32, i32, i32, i32, vp, C.c_float, i32, vp, vp]),
            "ds_csr_scatter": (C.c_int, [i32, vp, vp, vp, i32, vp, vp]),
            "ds_stream_create": (C.c_int, [vp, vp]), "ds_stream_destroy": (None, [vp]),
            "ds_stream_begin": (C.c_int, [vp, i32, vp, vp, i32]),
            "ds_stream_upload": (C.c_int, [vp, i32, i32, vp, vp, vp]),
            "ds_stream_dock": (C.c_int, [vp, vp, vp, vp, i32, vp, vp]),
            "ds_stream_download": (C.c_int, [vp, vp, vp]),
            "ds_set_host_threads": (C.c_int, [i32]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.ds_abi_version() != 1:
            raise NativeUnavailable("libdockscreen ABI mismatch")
        _lib = L
        return L


def pinned_empty(shape, dtype) -> np.ndarray:
    """A numpy array in pinned host memory (ds_host_alloc); ds_dock DMAs such arrays directly."""
    dtype = np.dtype(dtype)
    count = int(np.prod(shape))
    nbytes = max(count * dtype.itemsize, 1)
    ptr = lib().ds_host_alloc(nbytes)
    if not ptr:
        raise MemoryError(f"ds_host_alloc({nbytes}) failed")
    buf = (C.c_char * nbytes).from_address(ptr)
    weakref.finalize(buf, lib().ds_host_free, ptr)
    return np.frombuffer(buf, dtype=dtype, count=count).reshape(shape)


class _PinnedPool:
    """Reusable page-locked blocks for per-call outputs (the batched engine's result arrays): an
    array from take() returns its block to the pool when the last view of it is gone, so a run
    whose previous report has been dropped reuses that report's pinned memory instead of page-
    locking (or page-faulting) hundreds of MB again.  At most keep_bytes stay pooled."""

    def __init__(self, keep_bytes: int = 2 << 30):
        self.keep = keep_bytes
        self.free: list = []      # (capacity, ptr), most recently returned last
        self.lock = threading.Lock()

    def take(self, shape, dtype) -> np.ndarray:
        dtype = np.dtype(dtype)
        count = int(np.prod(shape))
        nbytes = max(count * dtype.itemsize, 1)
        ptr = cap = None
        with self.lock:
            fits = [k for k, (c, _) in enumerate(self.free) if nbytes <= c <= 2 * nbytes + (1 << 20)]
            if fits:
                k = min(fits, key=lambda k: self.free[k][0])
                cap, ptr = self.free.pop(k)
        if ptr is None:
            cap = nbytes + nbytes // 4
            ptr = lib().ds_host_alloc(cap)
            if not ptr:
                raise MemoryError(f"ds_host_alloc({cap}) failed")
        buf = (C.c_char * nbytes).from_address(ptr)
        weakref.finalize(buf, self._give_back, cap, ptr)
        return np.frombuffer(buf, dtype=dtype, count=count).reshape(shape)

    def _give_back(self, cap: int, ptr: int):
        with self.lock:
            self.free.append((cap, ptr))
            drop = []
            while sum(c for c, _ in self.free) > self.keep:
                drop.append(self.free.pop(0))
        for _, p in drop:
            lib().ds_host_free(p)


_OUT_POOL = _PinnedPool()


def pooled_pinned_empty(shape, dtype) -> np.ndarray:
    """pinned_empty from the reusable output pool (see _PinnedPool)."""
    return _OUT_POOL.take(shape, dtype)


def pinned_copy(a: np.ndarray) -> np.ndarray:
    out = pinned_empty(a.shape, a.dtype)
    out[...] = a
    return out


def check(rc: int):
    if rc != DS_OK:
        msg = lib().ds_last_error().decode(errors="replace")
        exc = ERRORS.get(rc)
        if exc is not None:
            raise exc(msg)
        if rc in (-9, -10):
            raise NativeUnavailable(msg)
        raise DsError(rc, msg)


def device_count() -> int:
    n = C.c_int(0)
    rc = lib().ds_device_count(C.byref(n))
    return int(n.value) if rc == DS_OK else 0


# ---- ligand batches --------------------------------------------------------------------
class GeneratedIds(_abc.Sequence):
    """The ids of generated ligands first .. first + n - 1 ("lig_<seed>_<index>"),
    materialised only on access: a 10M-ligand screen never builds 10M Python strings, and
    id_blob() makes the packed id bytes natively (ds_generated_ids)."""

    def __init__(self, seed: int, first: int, n: int):
        self.seed, self.first, self.n = int(seed), int(first), int(n)

    def __len__(self) -> int:
        return self.n

    def __getitem__(self, i):
        if isinstance(i, slice):
            lo, hi, step = i.indices(self.n)
            if step != 1:
                return [self[k] for k in range(lo, hi, step)]
            return GeneratedIds(self.seed, self.first + lo, max(hi - lo, 0))
        i = int(i)
        if i < 0:
            i += self.n
        if not 0 <= i < self.n:
            raise IndexError(i)
        return f"lig_{self.seed}_{self.first + i}"

    def __eq__(self, other) -> bool:
        return list(self) == list(other) if isinstance(other, (list, tuple, GeneratedIds)) else NotImplemented

    def id_blob(self):
        off = np.zeros(self.n + 1, np.int64)
        check(lib().ds_generated_ids(self.seed, self.first, self.n, None, _p(off)))
        buf = np.zeros(max(int(off[-1]), 1), np.uint8)
        check(lib().ds_generated_ids(self.seed, self.first, self.n, _p(buf), _p(off)))
        return buf[:int(off[-1])].tobytes(), off


@dataclass
class LigandBatch:
    """CSR ligand batch in the reference's terms (absolute Å coordinates, element codes,
    bonds, fragments with moving-mask bitsets) plus the ids."""
    atom_off: np.ndarray      # int32 [n+1]
    atom_xyz: np.ndarray      # float32 [atoms, 3]
    atom_type: np.ndarray     # uint8 [atoms]
    bond_off: np.ndarray      # int32 [n+1]
    bonds: np.ndarray         # int32 [bonds, 2]
    frag_off: np.ndarray      # int32 [n+1]
    frag_axis: np.ndarray     # int32 [frags, 2]
    frag_mask: np.ndarray     # uint32 [frags, 5]
    ids: List[str]

    @property
    def n(self) -> int:
        return len(self.atom_off) - 1

    def n_atoms(self) -> np.ndarray:
        return np.diff(self.atom_off)

    def n_frags(self) -> np.ndarray:
        return np.diff(self.frag_off)

    def id_bytes(self):
        if isinstance(self.ids, GeneratedIds):
            return self.ids.id_blob()
        enc = [s.encode() for s in self.ids]
        off = np.zeros(len(enc) + 1, dtype=np.int64)
        off[1:] = np.cumsum([len(e) for e in enc])
        return b"".join(enc), off

    def slice(self, lo: int, hi: int) -> "LigandBatch":
        """Ligands [lo, hi) as a new batch (array slices, no per-ligand objects)."""
        a0, a1 = int(self.atom_off[lo]), int(self.atom_off[hi])
        b0, b1 = int(self.bond_off[lo]), int(self.bond_off[hi])
        f0, f1 = int(self.frag_off[lo]), int(self.frag_off[hi])
        return LigandBatch(self.atom_off[lo:hi + 1] - a0, self.atom_xyz[a0:a1], self.atom_type[a0:a1],
                           self.bond_off[lo:hi + 1] - b0, self.bonds[b0:b1], self.frag_off[lo:hi + 1] - f0,
                           self.frag_axis[f0:f1], self.frag_mask[f0:f1],
                           self.ids[lo:hi] if isinstance(self.ids, GeneratedIds) else list(self.ids[lo:hi]))

    def subset(self, idx: Sequence[int]) -> "LigandBatch":
        return LigandBatch.from_ligands([self.ligand(int(i)) for i in idx])

    def ligand(self, i: int) -> model.Ligand:
        a0, a1 = int(self.atom_off[i]), int(self.atom_off[i + 1])
        atoms = tuple(model.Atom.of(*self.atom_xyz[k], int(self.atom_type[k])) for k in range(a0, a1))
        b0, b1 = int(self.bond_off[i]), int(self.bond_off[i + 1])
        bonds = tuple((int(a), int(b)) for a, b in self.bonds[b0:b1])
        frags = []
        for f in range(int(self.frag_off[i]), int(self.frag_off[i + 1])):
            bits = self.frag_mask[f]
            mask = frozenset(k for k in range(a1 - a0) if (int(bits[k >> 5]) >> (k & 31)) & 1)
            frags.append(model.Fragment(int(self.frag_axis[f, 0]), int(self.frag_axis[f, 1]), mask))
        return model.Ligand(self.ids[i], atoms, bonds, tuple(frags))

    def to_ligands(self) -> List[model.Ligand]:
        return [self.ligand(i) for i in range(self.n)]

    @staticmethod
    def from_ligands_validated(ligands: Sequence[model.Ligand]) -> Tuple["LigandBatch", np.ndarray]:
        """Flatten the reference's Ligand objects in bulk and run validate_ligand on
        all of them natively (ds_validate_ligands, all host cores).  Returns the batch of the valid
        ligands (input order) and the DS_ERR_* code of every input ligand (0 = valid)."""
        import itertools
        n = len(ligands)
        na = np.fromiter((len(l.atoms) for l in ligands), np.int64, n)
        nb = np.fromiter((len(l.bonds) for l in ligands), np.int64, n)
        nf = np.fromiter((len(l.fragments) for l in ligands), np.int64, n)
        atoms = [a for l in ligands for a in l.atoms]
        xyz = np.fromiter(itertools.chain.from_iterable(a.position for a in atoms), np.float64,
                          3 * len(atoms)).reshape(-1, 3)
        typ = np.fromiter((a.element_type for a in atoms), np.int64, len(atoms))
        heavy = np.fromiter((a.is_heavy for a in atoms), np.uint8, len(atoms))
        bonds = np.fromiter(itertools.chain.from_iterable(b for l in ligands for b in l.bonds), np.int64,
                            2 * int(nb.sum())).reshape(-1, 2)
        frags = [f for l in ligands for f in l.fragments]
        axis = np.fromiter(itertools.chain.from_iterable((f.axis_begin, f.axis_end) for f in frags), np.int64,
                           2 * len(frags)).reshape(-1, 2)
        mlen = np.fromiter((len(f.moving_mask) for f in frags), np.int64, len(frags))
        mv = np.fromiter(itertools.chain.from_iterable(f.moving_mask for f in frags), np.int64, int(mlen.sum()))
        off = lambda c: np.concatenate([[0], np.cumsum(c)]).astype(np.int64)
        ao, bo, fo, mo = off(na), off(nb), off(nf), off(mlen)
        i32 = lambda a: np.ascontiguousarray(np.clip(a, -2**31, 2**31 - 1).astype(np.int32))
        codes = np.zeros(max(n, 1), np.int32)
        if n > 0 and (ao[-1] >= 2**31 or bo[-1] >= 2**31 or fo[-1] >= 2**31):
            raise ValueError("batch too large for one validation call")
        if n:
            # _p passes raw addresses: every array must stay referenced until the call returns
            keep = [i32(ao), np.ascontiguousarray(typ), heavy, i32(bo), i32(bonds).reshape(-1), i32(fo),
                    i32(axis).reshape(-1), np.ascontiguousarray(mo), np.ascontiguousarray(mv), codes]
            check(lib().ds_validate_ligands(n, *[_p(x) for x in keep]))
        codes = codes[:n]
        okm = codes == 0
        ok = np.nonzero(okm)[0]
        # the valid ligands' arrays, in input order (boolean masks repeated per atom / bond / fragment)
        ka = np.nonzero(np.repeat(okm, na))[0]
        kb = np.nonzero(np.repeat(okm, nb))[0]
        fok = np.repeat(okm, nf)
        kf = np.nonzero(fok)[0]
        mask = np.zeros((len(kf), MASK_WORDS), np.uint32)
        if len(kf):
            cnt = mlen[kf]
            rows = np.repeat(np.arange(len(kf)), cnt)
            vals = mv[np.repeat(fok, mlen)]
            np.bitwise_or.at(mask, (rows, vals >> 5), (np.uint32(1) << (vals & 31).astype(np.uint32)))
        o32 = lambda c: np.concatenate([[0], np.cumsum(c)]).astype(np.int32)
        batch = LigandBatch(o32(na[ok]), xyz[ka].astype(np.float32), typ[ka].astype(np.uint8), o32(nb[ok]),
                            bonds[kb].astype(np.int32).reshape(-1, 2), o32(nf[ok]), axis[kf].astype(np.int32).reshape(-1, 2),
                            mask, [ligands[i].id for i in ok])
        return batch, codes

    @staticmethod
    def from_ligands(ligands: Sequence[model.Ligand]) -> "LigandBatch":
        n = len(ligands)
        na = np.array([len(l.atoms) for l in ligands], dtype=np.int32)
        nb = np.array([len(l.bonds) for l in ligands], dtype=np.int32)
        nf = np.array([len(l.fragments) for l in ligands], dtype=np.int32)
        off = lambda c: np.concatenate([[0], np.cumsum(c)]).astype(np.int32)
        xyz = np.zeros((int(na.sum()), 3), dtype=np.float32)
        typ = np.zeros(int(na.sum()), dtype=np.uint8)
        bonds = np.zeros((int(nb.sum()), 2), dtype=np.int32)
        axis = np.zeros((int(nf.sum()), 2), dtype=np.int32)
        mask = np.zeros((int(nf.sum()), MASK_WORDS), dtype=np.uint32)
        ao, bo, fo = off(na), off(nb), off(nf)
        for i, l in enumerate(ligands):
            if len(l.atoms) > model.MAX_ATOMS:
                raise model.TooManyAtoms(f"{l.id}: {len(l.atoms)} atoms")
            if l.atoms:
                xyz[ao[i]:ao[i + 1]] = np.array([a.position for a in l.atoms], dtype=np.float32)
                typ[ao[i]:ao[i + 1]] = [a.element_type for a in l.atoms]
            if l.bonds:
                bonds[bo[i]:bo[i + 1]] = np.array(l.bonds, dtype=np.int32)
            for k, f in enumerate(l.fragments):
                axis[fo[i] + k] = (f.axis_begin, f.axis_end)
                for m in f.moving_mask:
                    if not (0 <= m < model.MAX_ATOMS):
                        raise model.IndexOutOfRange(f"{l.id}: mask index {m}")
                    mask[fo[i] + k, m >> 5] |= np.uint32(1 << (m & 31))
        return LigandBatch(ao, xyz, typ, bo, bonds, fo, axis, mask, [l.id for l in ligands])


@dataclass
class PackedBatch:
    """The ds_batch_desc layout (centred coordinates, fragment records, id hashes)."""
    n: int
    atom_off: np.ndarray
    atom_xyzt: np.ndarray     # float32 [atoms, 4]
    frag_off: np.ndarray
    frag_desc: np.ndarray     # uint32 [frags, 8]
    id_hash: np.ndarray       # uint64 [n]
    centroid: np.ndarray      # float32 [n, 3]

    def desc(self) -> BatchDesc:
        d = BatchDesc()
        d.n_ligands = self.n
        d.atom_off = _p(self.atom_off)
        d.atom_xyzt = _p(self.atom_xyzt)
        d.frag_off = _p(self.frag_off)
        d.frag_desc = _p(self.frag_desc)
        d.id_hash = _p(self.id_hash)
        return d


def pack(batch: LigandBatch, pinned: bool = False) -> PackedBatch:
    """Validate + pack (ds_pack_ligands): c0 = f32(f64 mean), d = p - c0 (DESIGN.md §3 P2).
    pinned=True places the packed arrays in page-locked memory (direct DMA by ds_dock)."""
    n = batch.n
    na, nf = int(batch.atom_off[-1]), int(batch.frag_off[-1])
    alloc = pinned_empty if pinned else (lambda s, d: np.empty(s, d))
    xyzt = alloc((max(na, 1), 4), np.float32)
    fdesc = alloc((max(nf, 1), FRAG_WORDS), np.uint32)
    idh = alloc(max(n, 1), np.uint64)
    cen = alloc((max(n, 1), 3), np.float32)
    ids, id_off = batch.id_bytes()
    idbuf = C.create_string_buffer(ids, max(len(ids), 1))
    bad = C.c_int32(-1)
    c = lambda a: np.ascontiguousarray(a)
    ao, xyz, typ = c(batch.atom_off.astype(np.int32)), c(batch.atom_xyz.astype(np.float32)), c(batch.atom_type.astype(np.uint8))
    fo, fax, fm = c(batch.frag_off.astype(np.int32)), c(batch.frag_axis.astype(np.int32)), c(batch.frag_mask.astype(np.uint32))
    if fax.size == 0:
        fax = np.zeros((1, 2), np.int32)
        fm = np.zeros((1, MASK_WORDS), np.uint32)
    rc = lib().ds_pack_ligands(n, _p(ao), _p(xyz), _p(typ), _p(fo), _p(fax), _p(fm), C.cast(idbuf, C.c_void_p),
                               _p(id_off), _p(xyzt), _p(fdesc), _p(idh), _p(cen), C.byref(bad))
    if rc != DS_OK:
        msg = lib().ds_last_error().decode(errors="replace")
        exc = ERRORS.get(rc, DsError)
        who = batch.ids[bad.value] if 0 <= bad.value < n else "?"
        raise exc(f"ligand {who}: invalid ({rc}) {msg}")
    if pinned:
        ao, fo = pinned_copy(ao), pinned_copy(fo)
    return PackedBatch(n, ao, xyzt, fo, fdesc, idh[:n] if n else idh[:0], cen)


# ---- pockets / tables ------------------------------------------------------------------
DEFAULT_BINS = ((2.0, 0.5), (4.0, 1.0), (6.0, 0.5), (8.0, 0.25))   # DESIGN.md §3 P11


@dataclass(frozen=True)
class InteractionTable:
    """16x16 symmetric weights + ascending (upper_bound, multiplier) bins."""
    table: np.ndarray
    bins: tuple = DEFAULT_BINS

    @staticmethod
    def default(seed: int = 11) -> "InteractionTable":
        t = np.zeros(256, dtype=np.float32)
        check(lib().ds_default_table(seed, _p(t)))
        return InteractionTable(t.reshape(16, 16), DEFAULT_BINS)

    @property
    def cutoff(self) -> float:
        return float(self.bins[-1][0])

    @staticmethod
    def load(path: str) -> "InteractionTable":
        """a plain-text table file — 16 lines of 16 reals (the symmetric weights), then
        one line per distance bin "upper multiplier" (ascending upper bounds, the last = the rescore
        cutoff).  Blank lines and '#' comments are ignored.  Malformed files raise ParseError."""
        rows, bins = [], []
        with open(path, encoding="ascii") as fh:
            for ln, line in enumerate(fh, 1):
                tok = line.split("#", 1)[0].split()
                if not tok:
                    continue
                try:
                    vals = [float(t) for t in tok]
                except ValueError as e:
                    raise model.ParseError(f"line {ln}: {e}") from e
                if len(rows) < 16:
                    if len(vals) != 16:
                        raise model.ParseError(f"line {ln}: table row needs 16 values, found {len(vals)}")
                    rows.append(vals)
                elif len(vals) == 2:
                    bins.append((vals[0], vals[1]))
                else:
                    raise model.ParseError(f"line {ln}: bin line needs 'upper multiplier'")
        if len(rows) < 16:
            raise model.ParseError(f"expected 16 table rows, found {len(rows)}")
        if not bins:
            raise model.ParseError("no distance bins")
        t = np.array(rows, np.float32)
        if not np.array_equal(t, t.T):
            raise model.ParseError("interaction table must be symmetric (SPEC.md:180)")
        ub = [b[0] for b in bins]
        if any(not (b > a) for a, b in zip(ub, ub[1:])) or not ub[0] > 0 or len(bins) > MAX_BINS:
            raise model.ParseError(f"bins must have 1..{MAX_BINS} ascending positive upper bounds")
        return InteractionTable(t, tuple((float(np.float32(u)), float(np.float32(m))) for u, m in bins))

    def save(self, path: str) -> None:
        """Write the SPEC.md:225 text format (float32 values, round-trip exact)."""
        with open(path, "w", encoding="ascii", newline="\n") as fh:
            for row in np.asarray(self.table, np.float32).reshape(16, 16):
                fh.write(" ".join(repr(float(v)) for v in row) + "\n")
            for u, m in self.bins:
                fh.write(f"{float(np.float32(u))!r} {float(np.float32(m))!r}\n")


class DevicePocket:
    """A pocket + interaction table uploaded to one context (shared read-only)."""

    def __init__(self, ctx: "Context", pocket: model.Pocket, table: InteractionTable):
        self.ctx, self.pocket, self.table = ctx, pocket, table
        xyz, typ = pocket.atom_arrays()
        self._keep = [pocket.grid_values, np.ascontiguousarray(xyz), np.ascontiguousarray(typ),
                      np.ascontiguousarray(table.table, dtype=np.float32).reshape(-1),
                      np.array([b[0] for b in table.bins], dtype=np.float32),
                      np.array([b[1] for b in table.bins], dtype=np.float32)]
        d = PocketDesc()
        for k in range(3):
            d.origin[k] = float(pocket.grid_origin[k])
            d.dims[k] = int(pocket.grid_dims[k])
        d.spacing = float(pocket.grid_spacing)
        d.n_atoms = len(typ)
        d.values, d.atom_xyz, d.atom_type, d.table, _, _ = (_p(a) for a in self._keep)
        d.n_bins = len(table.bins)
        d.bin_ub, d.bin_mult = _p(self._keep[4]), _p(self._keep[5])
        h = C.c_void_p()
        check(lib().ds_pocket_create(ctx.handle, C.byref(d), C.byref(h)))
        self.handle = h

    def close(self):
        if self.handle:
            lib().ds_pocket_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def config_c(cfg: model.DockConfig, seed: int = 0) -> DockConfigC:
    c = DockConfigC()
    c.restarts_n, c.rescore_top_k = cfg.restarts_n, cfg.rescore_top_k
    c.alignment_step_deg, c.torsion_step_deg = cfg.alignment_step_deg, cfg.torsion_step_deg
    c.bump_distance, c.similarity_rmsd, c.rescore_cutoff = cfg.bump_distance, cfg.similarity_rmsd, cfg.rescore_cutoff
    c.early_exit = 1 if cfg.early_exit else 0
    c.seed = int(seed)
    return c


@dataclass
class DockOutput:
    results: np.ndarray               # RESULT_DTYPE [n]
    best_coords: Optional[np.ndarray]  # float32 [atoms, 3]
    best_torsion: Optional[np.ndarray]  # uint8 [frags]
    restarts: Optional[np.ndarray]     # RESTART_DTYPE [n, N]
    restart_torsion: Optional[np.ndarray]  # uint8 [frags, N]
    stats: Stats


class OutputBuffers:
    """Reusable (pinned by default) result buffers for repeated ds_dock calls on one batch shape."""

    def __init__(self, packed: PackedBatch, pinned: bool = True):
        alloc = pinned_empty if pinned else (lambda s, d: np.zeros(s, d))
        n = packed.n
        na, nf = int(packed.atom_off[-1]) if n else 0, int(packed.frag_off[-1]) if n else 0
        self.results = alloc(max(n, 1), RESULT_DTYPE)
        self.best_coords = alloc((max(na, 1), 3), np.float32)
        self.best_torsion = alloc(max(nf, 1), np.uint8)


class Context:
    """ds_ctx: one CUDA stream + workspaces on one device."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib().ds_create(int(device), C.byref(h)))
        self.handle = h
        self.device = device

    def reserve(self, cfg: model.DockConfig, max_ligands: int = 1, max_atoms: int = model.MAX_ATOMS,
                max_frags: int = model.MAX_ATOMS - 2):
        """Allocate the worst-case workspace once: one ligand of 160 atoms by default."""
        check(lib().ds_ctx_reserve(self.handle, int(max_ligands), int(max_atoms), int(max_frags),
                                   C.byref(config_c(cfg))))

    def alloc_count(self) -> int:
        n = C.c_int64(0)
        check(lib().ds_ctx_alloc_count(self.handle, C.byref(n)))
        return int(n.value)

    def pocket(self, pocket: model.Pocket, table: Optional[InteractionTable] = None) -> DevicePocket:
        return DevicePocket(self, pocket, table or InteractionTable.default())

    def build_pocket_grid(self, atom_xyz: np.ndarray, spacing: float, padding: float):
        """build_pocket's grid on this context's device, bit-identical to the host build.
        Returns (origin, dims, values x-fastest int32, kernel ms)."""
        xyz = np.ascontiguousarray(atom_xyz, dtype=np.float32).reshape(-1, 3)
        origin = (C.c_float * 3)()
        dims = (C.c_int32 * 3)()
        check(lib().ds_build_pocket_grid(_p(xyz), len(xyz), float(spacing), float(padding), origin, dims, None))
        vals = np.zeros(int(dims[0]) * int(dims[1]) * int(dims[2]), np.int32)
        ms = C.c_float(0.0)
        check(lib().ds_build_pocket_grid_device(self.handle, _p(xyz), len(xyz), float(spacing), float(padding), origin,
                                                dims, _p(vals), C.byref(ms)))
        return tuple(float(o) for o in origin), tuple(int(d) for d in dims), vals, float(ms.value)

    def dock(self, dpocket: DevicePocket, packed: PackedBatch, cfg: model.DockConfig, seed: int = 0,
             family: int = FAMILY_BATCHED, coords: bool = True, detail: bool = False,
             buffers: Optional["OutputBuffers"] = None) -> DockOutput:
        """ds_dock on host buffers.  `buffers` (e.g. pinned OutputBuffers) are reused if given."""
        n, N = packed.n, cfg.restarts_n
        na, nf = int(packed.atom_off[-1]) if n else 0, int(packed.frag_off[-1]) if n else 0
        if buffers is not None:
            res, bc, bt = buffers.results, (buffers.best_coords if coords else None), buffers.best_torsion
        else:
            res = np.zeros(max(n, 1), dtype=RESULT_DTYPE)
            bc = np.zeros((max(na, 1), 3), dtype=np.float32) if coords else None
            bt = np.zeros(max(nf, 1), dtype=np.uint8)
        rr = np.zeros((max(n, 1), N), dtype=RESTART_DTYPE) if detail else None
        rt = np.zeros((max(nf, 1), N), dtype=np.uint8) if detail else None
        out = Outputs(_p(res), _p(bc), _p(bt), _p(rr), _p(rt))
        st = Stats()
        ccfg = config_c(cfg, seed)
        check(lib().ds_dock(self.handle, dpocket.handle, C.byref(packed.desc()), C.byref(ccfg), int(family),
                            C.byref(out), C.byref(st)))
        return DockOutput(res[:n], bc[:na] if bc is not None else None, bt[:nf],
                          rr[:n] if rr is not None else None, rt[:nf] if rt is not None else None, st)

    def close(self):
        # pockets cached on this context (docking.PocketCache) are released first, deterministically,
        # instead of being left to the cyclic GC in arbitrary order
        cache = self.__dict__.pop("_pocket_cache", None)
        if cache:
            for hit in cache.values():
                hit[2].close()
        if getattr(self, "handle", None):
            lib().ds_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


class EngineStream:
    """ds_stream: the packed ligand stream of a batched-engine run kept on one device.
    begin() sizes it, producers upload() the ranges they packed, dispatchers dock() index lists of
    stream ligands on their own contexts, download() returns every ligand's outputs."""

    def __init__(self, ctx: Context):
        h = C.c_void_p()
        check(lib().ds_stream_create(ctx.handle, C.byref(h)))
        self.handle, self.device = h, ctx.device
        self._atom_off = self._frag_off = None

    def begin(self, atom_off: np.ndarray, frag_off: np.ndarray, restarts: int):
        self._atom_off = np.ascontiguousarray(atom_off, np.int32)
        self._frag_off = np.ascontiguousarray(frag_off, np.int32)
        check(lib().ds_stream_begin(self.handle, len(self._atom_off) - 1, _p(self._atom_off), _p(self._frag_off),
                                    int(restarts)))

    def upload(self, lo: int, hi: int, xyzt: np.ndarray, fdesc: np.ndarray, idh: np.ndarray):
        check(lib().ds_stream_upload(self.handle, int(lo), int(hi), _p(xyzt), _p(fdesc), _p(idh)))

    def dock(self, ctx: Context, dpocket: "DevicePocket", sel: np.ndarray, cfg: model.DockConfig,
             seed: int = 0) -> Stats:
        sel = np.ascontiguousarray(sel, np.int32)
        st = Stats()
        ccfg = config_c(cfg, seed)
        check(lib().ds_stream_dock(ctx.handle, dpocket.handle, self.handle, _p(sel), len(sel), C.byref(ccfg),
                                   C.byref(st)))
        return st

    def download(self, ctx: Context, results: np.ndarray, best_coords: Optional[np.ndarray],
                 best_torsion: Optional[np.ndarray]):
        out = Outputs(_p(results), _p(best_coords), _p(best_torsion), None, None)
        check(lib().ds_stream_download(ctx.handle, self.handle, C.byref(out)))

    def close(self):
        if getattr(self, "handle", None):
            lib().ds_stream_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ResidentBatch:
    """A packed batch kept in device memory (kernel-only timing, bench.py `value`)."""

    def __init__(self, ctx: Context, packed: Optional[PackedBatch], handle=None, n: int = 0,
                 atom_off: Optional[np.ndarray] = None, frag_off: Optional[np.ndarray] = None):
        if handle is None:
            handle = C.c_void_p()
            check(lib().ds_batch_upload(ctx.handle, C.byref(packed.desc()), C.byref(handle)))
            n, atom_off, frag_off = packed.n, packed.atom_off, packed.frag_off
        self.ctx, self.packed, self.handle, self.n = ctx, packed, handle, n
        self.atom_off, self.frag_off = atom_off, frag_off
        self.generate_ms = 0.0

    @classmethod
    def generated(cls, ctx: Context, seed: int, first_index: int, shapes: np.ndarray) -> "ResidentBatch":
        """Device-side ingest (ds_generate_resident): ligands first_index .. + len(shapes) of the
        synthetic dataset generated and packed on the GPU — the same arrays as
        ResidentBatch(ctx, pack(io.generate_batch(shapes, seed, first_index)))."""
        shapes = np.ascontiguousarray(np.asarray(shapes, np.int32).reshape(-1, 2))
        h, ms = C.c_void_p(), C.c_float(0.0)
        check(lib().ds_generate_resident(ctx.handle, int(seed), int(first_index), len(shapes), _p(shapes), C.byref(h),
                                         C.byref(ms)))
        n = len(shapes)
        ao, bo, fo = (np.zeros(n + 1, np.int32) for _ in range(3))
        check(lib().ds_generate_ligands(int(seed), int(first_index), n, _p(shapes), _p(ao), _p(bo), _p(fo),
                                        None, None, None, None, None))
        rb = cls(ctx, None, handle=h, n=n, atom_off=ao, frag_off=fo)
        rb.generate_ms = float(ms.value)
        return rb

    def read_inputs(self):
        """(atom_xyzt [atoms, 4] f32, frag_desc [frags, 8] u32, id_hash [n] u64) as resident."""
        na, nf = int(self.atom_off[-1]), int(self.frag_off[-1])
        xyzt = np.zeros((max(na, 1), 4), np.float32)
        fd = np.zeros((max(nf, 1), FRAG_WORDS), np.uint32)
        idh = np.zeros(max(self.n, 1), np.uint64)
        check(lib().ds_batch_read_inputs(self.ctx.handle, self.handle, _p(xyzt), _p(fd), _p(idh)))
        return xyzt[:na], fd[:nf], idh[:self.n]

    def dock(self, dpocket: DevicePocket, cfg: model.DockConfig, seed: int = 0, family: int = FAMILY_BATCHED) -> Stats:
        st = Stats()
        ccfg = config_c(cfg, seed)
        check(lib().ds_dock_resident(self.ctx.handle, dpocket.handle, self.handle, C.byref(ccfg), int(family),
                                     C.byref(st)))
        return st

    def download(self, coords: bool = False, torsion: bool = False, results: Optional[np.ndarray] = None,
                 best_torsion: Optional[np.ndarray] = None):
        """The result records; with coords / torsion also the best poses (Å) and the best pose's
        per-fragment torsion indices: (records, coords or None, torsion or None)."""
        na, nf = int(self.atom_off[-1]) if self.n else 0, int(self.frag_off[-1]) if self.n else 0
        res = results if results is not None else np.zeros(max(self.n, 1), dtype=RESULT_DTYPE)
        bc = np.zeros((max(na, 1), 3), np.float32) if coords else None
        bt = (best_torsion if best_torsion is not None else np.zeros(max(nf, 1), np.uint8)) if torsion else None
        out = Outputs(_p(res), _p(bc), _p(bt), None, None)
        check(lib().ds_batch_download(self.ctx.handle, self.handle, C.byref(out)))
        if not coords and not torsion:
            return res[:self.n]
        return res[:self.n], (bc[:na] if bc is not None else None), (bt[:nf] if bt is not None else None)

    def close(self):
        if self.handle:
            lib().ds_batch_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
