"""core-model: the reference's domain records.

Immutable records shared by every other module.  Field names, defaults and the
validation errors follow SPEC.md's `core-model` module; `validate_ligand` checks the
invariants of SPEC.md:26-47 (including the bond-cut rule of SPEC.md:38).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Sequence, Tuple

import numpy as np

MAX_ATOMS = 160          # SPEC.md:44 (largest bucket bound)
N_TYPES = 16             # SPEC.md:95 closed element enumeration
HYDROGEN = 0             # DESIGN.md §3 P16 (SPEC.md:27-30 leaves the code open)


# ---- errors -------------------------------------------
class DockscreenError(Exception):
    """Base class of the reference's named errors."""


class TooManyAtoms(DockscreenError):
    pass


class MalformedFragment(DockscreenError):
    pass


class IndexOutOfRange(DockscreenError):
    pass


class DegenerateAxis(DockscreenError):
    pass


class NoValidPose(DockscreenError):
    pass


class EmptyPocket(DockscreenError):
    pass


class InfeasibleShape(DockscreenError):
    pass


class ParseError(DockscreenError):
    pass


class ValidationError(DockscreenError):
    pass


# ---- records ---------------------------------------------------------------------------
@dataclass(frozen=True)
class Atom:
    """SPEC.md:26-31."""
    position: Tuple[float, float, float]
    element_type: int
    is_heavy: bool = True

    @staticmethod
    def of(x: float, y: float, z: float, element_type: int) -> "Atom":
        return Atom((float(x), float(y), float(z)), int(element_type), int(element_type) != HYDROGEN)


@dataclass(frozen=True)
class Fragment:
    """rotatable bond axis_begin->axis_end and the moving side."""
    axis_begin: int
    axis_end: int
    moving_mask: frozenset


@dataclass(frozen=True)
class Ligand:
    """SPEC.md:41-47."""
    id: str
    atoms: Tuple[Atom, ...]
    bonds: Tuple[Tuple[int, int], ...] = ()
    fragments: Tuple[Fragment, ...] = ()

    @property
    def heavy_atom_count(self) -> int:
        return sum(1 for a in self.atoms if a.is_heavy)

    def coords(self) -> np.ndarray:
        return np.array([a.position for a in self.atoms], dtype=np.float32).reshape(-1, 3)

    def types(self) -> np.ndarray:
        return np.array([a.element_type for a in self.atoms], dtype=np.uint8)


@dataclass(frozen=True)
class Pocket:
    """SPEC.md:49-54.  grid_values is x-fastest, stored as a flat int32 array."""
    grid_origin: Tuple[float, float, float]
    grid_spacing: float
    grid_dims: Tuple[int, int, int]
    grid_values: np.ndarray = field(repr=False, compare=False)
    pocket_atoms: Tuple[Atom, ...] = ()

    def __post_init__(self):
        vals = np.ascontiguousarray(np.asarray(self.grid_values, dtype=np.int32).reshape(-1))
        object.__setattr__(self, "grid_values", vals)
        nx, ny, nz = (int(d) for d in self.grid_dims)
        if min(nx, ny, nz) < 1 or vals.size != nx * ny * nz:
            raise ValueError("grid_values length must equal the product of grid_dims")
        if not self.grid_spacing > 0:
            raise ValueError("grid_spacing must be > 0")

    def atom_arrays(self):
        xyz = np.array([a.position for a in self.pocket_atoms], dtype=np.float32).reshape(-1, 3)
        typ = np.array([a.element_type for a in self.pocket_atoms], dtype=np.uint8)
        return xyz, typ


@dataclass(frozen=True)
class DockConfig:
    """SPEC.md:63-68 (defaults as printed)."""
    restarts_n: int = 8
    rescore_top_k: int = 4
    alignment_step_deg: int = 12
    torsion_step_deg: int = 36
    bump_distance: float = 0.8
    similarity_rmsd: float = 1.0
    rescore_cutoff: float = 8.0
    early_exit: bool = True

    def __post_init__(self):
        if self.restarts_n < 1 or self.rescore_top_k < 1:
            raise ValueError("restarts_n and rescore_top_k must be positive")
        if self.rescore_top_k > self.restarts_n:
            raise ValueError("rescore_top_k must be <= restarts_n")
        if 360 % self.alignment_step_deg or 360 % self.torsion_step_deg:
            raise ValueError("360 must be divisible by the angle steps")
        if not (self.bump_distance > 0 and self.similarity_rmsd > 0 and self.rescore_cutoff > 0):
            raise ValueError("distances must be positive")


@dataclass
class Counters:
    """SPEC.md:75-78 (merged by summation)."""
    poses_scored: int = 0
    bump_checks: int = 0
    bump_early_exits: int = 0
    batches_dispatched: int = 0
    batch_fill_ratio_sum: float = 0.0

    def merge(self, other: "Counters") -> "Counters":
        self.poses_scored += other.poses_scored
        self.bump_checks += other.bump_checks
        self.bump_early_exits += other.bump_early_exits
        self.batches_dispatched += other.batches_dispatched
        self.batch_fill_ratio_sum += other.batch_fill_ratio_sum
        return self


@dataclass(frozen=True)
class Pose:
    """SPEC.md:56-61.  Extra fields record the selected indices (bit-exact parity targets)."""
    coordinates: np.ndarray = field(repr=False, compare=False)
    geometric_score: int
    chemical_score: float
    restart_index: int
    valid: bool
    align_indices: Tuple[int, int] = (0, 0)
    torsion_indices: Tuple[int, ...] = ()
    chem_fx: int = 0


@dataclass(frozen=True)
class DockResult:
    """SPEC.md:70-73.  best_pose is None iff the result is flagged (error set)."""
    ligand_id: str
    best_pose: Optional[Pose]
    counters: Counters
    error: Optional[str] = None

    @property
    def ok(self) -> bool:
        return self.best_pose is not None


# ---- validation --------------------------------------------------------
def _components_without(n: int, bonds: Sequence[Tuple[int, int]], cut: Tuple[int, int]):
    parent = list(range(n))

    def find(x):
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    cut_set = {cut, (cut[1], cut[0])}
    for (a, b) in bonds:
        if (a, b) in cut_set:
            continue
        ra, rb = find(a), find(b)
        if ra != rb:
            parent[ra] = rb
    return [find(i) for i in range(n)]


def validate_ligand(ligand: Ligand) -> Ligand:
    """Return the ligand iff every Ligand/Fragment invariant holds."""
    n = len(ligand.atoms)
    if n > MAX_ATOMS:
        raise TooManyAtoms(f"{ligand.id}: {n} atoms > {MAX_ATOMS}")
    if n < 1:
        raise IndexOutOfRange(f"{ligand.id}: ligand has no atoms")
    for a in ligand.atoms:
        if not (0 <= a.element_type < N_TYPES):
            raise IndexOutOfRange(f"{ligand.id}: element_type {a.element_type} outside 0..15")
        if a.is_heavy != (a.element_type != HYDROGEN):
            raise MalformedFragment(f"{ligand.id}: is_heavy inconsistent with element_type")
    for (a, b) in ligand.bonds:
        if not (0 <= a < n and 0 <= b < n):
            raise IndexOutOfRange(f"{ligand.id}: bond ({a},{b}) out of range")
    for f in ligand.fragments:
        if not (0 <= f.axis_begin < n and 0 <= f.axis_end < n):
            raise IndexOutOfRange(f"{ligand.id}: fragment axis out of range")
        if any(not (0 <= i < n) for i in f.moving_mask):
            raise IndexOutOfRange(f"{ligand.id}: moving_mask index out of range")
        if f.axis_begin == f.axis_end or f.axis_begin in f.moving_mask or f.axis_end in f.moving_mask:
            raise MalformedFragment(f"{ligand.id}: axis atoms must be distinct and outside the mask")
        if not f.moving_mask or len(f.moving_mask) >= n:
            raise MalformedFragment(f"{ligand.id}: moving_mask must be a non-empty proper subset")
        bond_set = {tuple(b) for b in ligand.bonds} | {(b[1], b[0]) for b in ligand.bonds}
        if (f.axis_begin, f.axis_end) not in bond_set:
            raise MalformedFragment(f"{ligand.id}: fragment axis is not a bond")
        comp = _components_without(n, ligand.bonds, (f.axis_begin, f.axis_end))
        cb, ce = comp[f.axis_begin], comp[f.axis_end]
        if cb == ce:
            raise MalformedFragment(f"{ligand.id}: removing the axis bond does not split the ligand")
        if len({c for c in comp}) != 2:
            raise MalformedFragment(f"{ligand.id}: cutting the axis bond must leave exactly two parts")
        part_b = {i for i in range(n) if comp[i] == cb} - {f.axis_begin, f.axis_end}
        part_e = {i for i in range(n) if comp[i] == ce} - {f.axis_begin, f.axis_end}
        if set(f.moving_mask) not in (part_b, part_e):
            raise MalformedFragment(f"{ligand.id}: moving_mask is not one side of the axis bond")
    return ligand
