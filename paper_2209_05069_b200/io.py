"""io: synthetic inputs and the `.ligq` / `.pock` text formats.

The generators run in libdockscreen's host code (C++, OpenMP) so a 10M-ligand screen
(BASELINE config 5) can be generated per shard on each rank; they are input makers, not the
timed hot path.
"""
from __future__ import annotations

import ctypes as C
from typing import Iterable, List, Optional, Sequence, Tuple

import numpy as np

from . import model
from .native import GeneratedIds, LigandBatch, InteractionTable, _p, check, lib, MASK_WORDS

SYNTH_POCKET = dict(n_atoms=200, seed=7, rmin=7.0, rmax=10.0, spacing=0.5, padding=4.0)


def generated_id(seed: int, index: int) -> str:
    buf = C.create_string_buffer(64)
    n = lib().ds_generated_id(int(seed), int(index), buf, 64)
    return buf.raw[:n].decode()


def generate_batch(shapes: np.ndarray, seed: int, first_index: int = 0) -> LigandBatch:
    """Packed generator: shapes[i] = (heavy, fragments) of ligand first_index + i."""
    shapes = np.ascontiguousarray(np.asarray(shapes, dtype=np.int32).reshape(-1, 2))
    n = len(shapes)
    ao = np.zeros(n + 1, np.int32)
    bo = np.zeros(n + 1, np.int32)
    fo = np.zeros(n + 1, np.int32)
    L = lib()
    check(L.ds_generate_ligands(int(seed), int(first_index), n, _p(shapes), _p(ao), _p(bo), _p(fo),
                                None, None, None, None, None))
    xyz = np.zeros((max(int(ao[-1]), 1), 3), np.float32)
    typ = np.zeros(max(int(ao[-1]), 1), np.uint8)
    bonds = np.zeros((max(int(bo[-1]), 1), 2), np.int32)
    axis = np.zeros((max(int(fo[-1]), 1), 2), np.int32)
    mask = np.zeros((max(int(fo[-1]), 1), MASK_WORDS), np.uint32)
    check(L.ds_generate_ligands(int(seed), int(first_index), n, _p(shapes), _p(ao), _p(bo), _p(fo),
                                _p(xyz), _p(typ), _p(bonds), _p(axis), _p(mask)))
    ids = GeneratedIds(seed, first_index, n)
    return LigandBatch(ao, xyz[:ao[-1]], typ[:ao[-1]], bo, bonds[:bo[-1]], fo, axis[:fo[-1]], mask[:fo[-1]], ids)


def mixed_shapes(count: int, seed: int, first_index: int = 0, heavy_range=(8, 40), frag_max: int = 20) -> np.ndarray:
    """(heavy, fragments) per ligand of the mixed datasets: heavy ~ U{8..40},
    F ~ U{0..min(20, heavy-2)}."""
    out = np.zeros((count, 2), np.int32)
    check(lib().ds_mixed_shapes(int(seed), int(first_index), int(count), int(heavy_range[0]), int(heavy_range[1]),
                                int(frag_max), _p(out)))
    return out


def generate_dataset_batch(heavy_atoms: int, fragments: int, count: int, seed: int, first_index: int = 0) -> LigandBatch:
    if fragments >= heavy_atoms - 1 and fragments > 0:
        raise model.InfeasibleShape(f"fragments={fragments} >= heavy_atoms-1={heavy_atoms - 1}")
    if heavy_atoms < 1 or heavy_atoms > model.MAX_ATOMS:
        raise model.InfeasibleShape(f"heavy_atoms={heavy_atoms}")
    shapes = np.tile(np.array([[heavy_atoms, fragments]], np.int32), (count, 1))
    return generate_batch(shapes, seed, first_index)


def generate_dataset(heavy_atoms: int, fragments: int, count: int, seed: int) -> List[model.Ligand]:
    """`count` chain ligands with exactly `heavy_atoms` heavy atoms and
    `fragments` rotatable bonds, 1-2 H per heavy atom (cap 160), self-avoiding 1.5 Å steps."""
    return generate_dataset_batch(heavy_atoms, fragments, count, seed).to_ligands()


def generate_mixed_batch(count: int, seed: int, first_index: int = 0, heavy_range=(8, 40), frag_max: int = 20) -> LigandBatch:
    return generate_batch(mixed_shapes(count, seed, first_index, heavy_range, frag_max), seed, first_index)


def pocket_atoms(n_atoms: int = 200, seed: int = 7, rmin: float = 7.0, rmax: float = 10.0) -> List[model.Atom]:
    xyz = np.zeros((n_atoms, 3), np.float32)
    typ = np.zeros(n_atoms, np.uint8)
    check(lib().ds_generate_pocket_atoms(int(seed), int(n_atoms), float(rmin), float(rmax), _p(xyz), _p(typ)))
    return [model.Atom.of(*xyz[i], int(typ[i])) for i in range(n_atoms)]


def build_pocket(pocket_atoms: Sequence[model.Atom], spacing: float, padding: float, ctx=None) -> model.Pocket:
    """grid over the atom bounding box + padding; node = round(10 g(d)),
    d = distance to the nearest pocket atom (DESIGN.md §3 P18).  With a `native.Context` the
    per-node scan runs on its GPU (bit-identical grid)."""
    if len(pocket_atoms) == 0:
        raise model.EmptyPocket("build_pocket needs at least one atom")
    if not spacing > 0:
        raise ValueError("spacing must be > 0")
    xyz = np.ascontiguousarray(np.array([a.position for a in pocket_atoms], dtype=np.float32))
    if ctx is not None:
        origin, dims, vals, _ = ctx.build_pocket_grid(xyz, spacing, padding)
        return model.Pocket(origin, float(np.float32(spacing)), dims, vals, tuple(pocket_atoms))
    origin = (C.c_float * 3)()
    dims = (C.c_int32 * 3)()
    L = lib()
    check(L.ds_build_pocket_grid(_p(xyz), len(pocket_atoms), float(spacing), float(padding), origin, dims, None))
    vals = np.zeros(int(dims[0]) * int(dims[1]) * int(dims[2]), np.int32)
    check(L.ds_build_pocket_grid(_p(xyz), len(pocket_atoms), float(spacing), float(padding), origin, dims, _p(vals)))
    return model.Pocket(tuple(float(o) for o in origin), float(np.float32(spacing)), tuple(int(d) for d in dims), vals,
                        tuple(pocket_atoms))


def synthetic_pocket(spacing: float = 0.5, **kw) -> model.Pocket:
    """The shared synthetic pocket of every BASELINE config: P=200, seed 7,
    shell 7-10 Å, spacing 0.5 Å (0.375 Å = the L2 variant), padding 4 Å."""
    p = dict(SYNTH_POCKET, spacing=spacing)
    p.update(kw)
    atoms = pocket_atoms(p["n_atoms"], p["seed"], p["rmin"], p["rmax"])
    return build_pocket(atoms, p["spacing"], p["padding"])


# ---- text formats -----------------------------------------------
def _fmt(x: float) -> str:
    return repr(float(np.float32(x)))


def write_ligand_file(path: str, ligands: Iterable[model.Ligand]) -> None:
    with open(path, "w", encoding="ascii", newline="\n") as fh:
        for l in ligands:
            fh.write(f"MOL {l.id}\n")
            for i, a in enumerate(l.atoms):
                fh.write(f"ATOM {i} {a.element_type} {_fmt(a.position[0])} {_fmt(a.position[1])} {_fmt(a.position[2])} "
                         f"{'heavy' if a.is_heavy else 'H'}\n")
            for (a, b) in l.bonds:
                fh.write(f"BOND {a} {b}\n")
            for f in l.fragments:
                fh.write("FRAG %d %d %s\n" % (f.axis_begin, f.axis_end, " ".join(str(m) for m in sorted(f.moving_mask))))
            fh.write("END\n")


def parse_ligand_file(path: str, skip_invalid: bool = False) -> List[model.Ligand]:
    """`.ligq` parser: MOL / ATOM / BOND / FRAG / END records; each molecule validated."""
    out: List[model.Ligand] = []
    cur = None
    with open(path, encoding="ascii") as fh:
        for ln, line in enumerate(fh, 1):
            tok = line.split()
            if not tok:
                continue
            try:
                if tok[0] == "MOL":
                    cur = dict(id=line.strip()[4:], atoms=[], bonds=[], frags=[], line=ln)
                elif cur is None:
                    raise model.ParseError(f"line {ln}: record outside MOL")
                elif tok[0] == "ATOM":
                    idx, typ = int(tok[1]), int(tok[2])
                    if idx != len(cur["atoms"]):
                        raise model.ParseError(f"line {ln}: atom index {idx} out of order")
                    x, y, z = (float(np.float32(float(t))) for t in tok[3:6])
                    heavy = tok[6] != "H"
                    cur["atoms"].append(model.Atom((x, y, z), typ, heavy))
                elif tok[0] == "BOND":
                    cur["bonds"].append((int(tok[1]), int(tok[2])))
                elif tok[0] == "FRAG":
                    cur["frags"].append(model.Fragment(int(tok[1]), int(tok[2]), frozenset(int(t) for t in tok[3:])))
                elif tok[0] == "END":
                    lig = model.Ligand(cur["id"], tuple(cur["atoms"]), tuple(cur["bonds"]), tuple(cur["frags"]))
                    try:
                        out.append(model.validate_ligand(lig))
                    except model.DockscreenError as e:
                        if not skip_invalid:
                            raise model.ValidationError(f"molecule {cur['id']} (line {cur['line']}): {e}") from e
                    cur = None
                else:
                    raise model.ParseError(f"line {ln}: unknown record {tok[0]!r}")
            except (ValueError, IndexError) as e:
                raise model.ParseError(f"line {ln}: {e}") from e
    if cur is not None:
        raise model.ParseError("missing END")
    return out


def parse_ligand_batch(path: str, skip_invalid: bool = False) -> LigandBatch:
    """Native `.ligq` reader (ds_ligq_parse): the same records, validation and errors as
    parse_ligand_file, parsed on all host cores straight into the packed CSR batch (host ingest at
    scale); no per-ligand Python objects until `.ligand(i)` / `.to_ligands()`."""
    with open(path, "rb") as fh:
        text = fh.read()
    L = lib()
    h = C.c_void_p()
    counts = (C.c_int64 * 6)()
    err = C.create_string_buffer(512)
    rc = L.ds_ligq_parse(text, len(text), int(bool(skip_invalid)), C.byref(h), counts, err, 512)
    if rc != 0:
        msg = err.value.decode(errors="replace")
        if rc == -12:
            raise model.ParseError(msg)
        raise model.ValidationError(msg)
    try:
        n, na, nb, nf, nid = (int(counts[k]) for k in range(5))
        ao, bo, fo = np.zeros(n + 1, np.int32), np.zeros(n + 1, np.int32), np.zeros(n + 1, np.int32)
        xyz, typ = np.zeros((max(na, 1), 3), np.float32), np.zeros(max(na, 1), np.uint8)
        bonds, axis = np.zeros((max(nb, 1), 2), np.int32), np.zeros((max(nf, 1), 2), np.int32)
        mask = np.zeros((max(nf, 1), MASK_WORDS), np.uint32)
        ids, id_off = C.create_string_buffer(max(nid, 1)), np.zeros(n + 1, np.int64)
        check(L.ds_ligq_fill(h, _p(ao), _p(xyz), _p(typ), _p(bo), _p(bonds), _p(fo), _p(axis), _p(mask),
                             C.cast(ids, C.c_void_p), _p(id_off)))
    finally:
        L.ds_ligq_free(h)
    raw = ids.raw
    names = [raw[id_off[i]:id_off[i + 1]].decode("ascii") for i in range(n)]
    return LigandBatch(ao, xyz[:na], typ[:na], bo, bonds[:nb], fo, axis[:nf], mask[:nf], names)


def write_pocket_file(path: str, pocket: model.Pocket) -> None:
    with open(path, "w", encoding="ascii", newline="\n") as fh:
        o = pocket.grid_origin
        fh.write(f"GRID {_fmt(o[0])} {_fmt(o[1])} {_fmt(o[2])} {_fmt(pocket.grid_spacing)} "
                 f"{pocket.grid_dims[0]} {pocket.grid_dims[1]} {pocket.grid_dims[2]}\n")
        vals = pocket.grid_values
        for k in range(0, len(vals), 32):
            fh.write(" ".join(str(int(v)) for v in vals[k:k + 32]) + "\n")
        for a in pocket.pocket_atoms:
            fh.write(f"PATOM {a.element_type} {_fmt(a.position[0])} {_fmt(a.position[1])} {_fmt(a.position[2])}\n")


def parse_pocket_file(path: str) -> model.Pocket:
    with open(path, encoding="ascii") as fh:
        head = fh.readline().split()
        if len(head) != 8 or head[0] != "GRID":
            raise model.ParseError("line 1: expected GRID ox oy oz spacing nx ny nz")
        o = tuple(float(np.float32(float(t))) for t in head[1:4])
        s = float(np.float32(float(head[4])))
        dims = tuple(int(t) for t in head[5:8])
        n = dims[0] * dims[1] * dims[2]
        vals: List[int] = []
        atoms: List[model.Atom] = []
        for ln, line in enumerate(fh, 2):
            tok = line.split()
            if not tok:
                continue
            if tok[0] == "PATOM":
                atoms.append(model.Atom.of(float(tok[2]), float(tok[3]), float(tok[4]), int(tok[1])))
            else:
                if atoms:
                    raise model.ParseError(f"line {ln}: grid values after PATOM records")
                vals.extend(int(t) for t in tok)
        if len(vals) != n:
            raise model.ParseError(f"expected {n} grid values, found {len(vals)}")
    return model.Pocket(o, s, dims, np.array(vals, np.int32), tuple(atoms))
