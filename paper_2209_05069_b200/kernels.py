"""kernels: the native slot `dockscreen.kernels._core` (pkg/setup.py:10-18) — the L2 ops of the
reference's `transform` and `scoring` modules on the B200.

Each op takes one pose (an [n, 3] array in Å) or a batch of poses ([P, n, 3]) and runs as one
device call through the C ABI (ds_op_*: include/dockscreen.h), with the numeric recipe of DESIGN.md
§3 — the same results, bit for bit, as oracle/ and as the docking kernels' inner loops.  rot_x / rot_y
are host functions (trig of integer degrees in f64, stored f32, P0: no device trig).

The Context comes from docking.thread_context (one per host thread and device).  There is no CPU
fallback: without libdockscreen.so or a CUDA device these raise.
"""
from __future__ import annotations

import ctypes as C
import math
from typing import Optional, Sequence, Tuple, Union

import numpy as np

from . import model
from .native import (CHEM_SCALE, STATUS_DEGENERATE_AXIS, DevicePocket, InteractionTable, MASK_WORDS, _p, check,
                     lib)

Coords = np.ndarray


def _trig(deg: int) -> Tuple[np.float32, np.float32]:
    rad = float(int(deg) % 360) * 0.017453292519943295   # P0
    return np.float32(math.cos(rad)), np.float32(math.sin(rad))


def rot_x(angle_deg: int) -> np.ndarray:
    """right-handed active rotation about x, f32 entries of f64 trig (P0)."""
    c, s = _trig(angle_deg)
    return np.array([[1, 0, 0], [0, c, -s], [0, s, c]], np.float32)


def rot_y(angle_deg: int) -> np.ndarray:
    """right-handed active rotation about y."""
    c, s = _trig(angle_deg)
    return np.array([[c, 0, s], [0, 1, 0], [-s, 0, c]], np.float32)


def _ctx(device: int = 0):
    from .docking import thread_context
    return thread_context(device)


def _poses(coords) -> Tuple[np.ndarray, bool]:
    a = np.ascontiguousarray(coords, np.float32)
    if a.ndim == 2:
        return a.reshape(1, -1, 3), True
    if a.ndim != 3 or a.shape[-1] != 3:
        raise ValueError("coords must be [n, 3] or [poses, n, 3]")
    return a, False


def _mask(frag: model.Fragment) -> np.ndarray:
    m = np.zeros(MASK_WORDS, np.uint32)
    for i in frag.moving_mask:
        if not 0 <= int(i) < 32 * MASK_WORDS:
            raise model.IndexOutOfRange(f"mask index {i}")
        m[int(i) >> 5] |= np.uint32(1 << (int(i) & 31))
    return m


def apply_rigid(coords: Coords, m, center, device: int = 0) -> np.ndarray:
    """p -> m (p - center) + center for every atom (batched: m [P, 3, 3], center [P, 3])."""
    P, single = _poses(coords)
    mm = np.ascontiguousarray(np.broadcast_to(np.asarray(m, np.float32).reshape(-1, 3, 3), (P.shape[0], 3, 3)))
    cc = np.ascontiguousarray(np.broadcast_to(np.asarray(center, np.float32).reshape(-1, 3), (P.shape[0], 3)))
    out = np.empty_like(P)
    check(lib().ds_op_apply_rigid(_ctx(device).handle, _p(P), P.shape[1], P.shape[0], _p(mm), _p(cc), _p(out)))
    return out[0] if single else out


def apply_torsion(coords: Coords, frag: model.Fragment, angle_deg: int, device: int = 0) -> np.ndarray:
    """rotate frag.moving_mask by angle_deg about axis_begin -> axis_end; other atoms
    bitwise unchanged; DegenerateAxis if the axis atoms coincide within 1e-9 Å."""
    P, single = _poses(coords)
    out = np.empty_like(P)
    st = np.zeros(P.shape[0], np.int32)
    check(lib().ds_op_apply_torsion(_ctx(device).handle, _p(P), P.shape[1], P.shape[0], int(frag.axis_begin),
                                    int(frag.axis_end), _p(_mask(frag)), int(angle_deg), _p(out), _p(st)))
    if (st == STATUS_DEGENERATE_AXIS).any():
        raise model.DegenerateAxis(f"axis atoms {frag.axis_begin}, {frag.axis_end} coincide "
                                   f"(pose {int(np.nonzero(st)[0][0])})")
    return out[0] if single else out


def _device_pocket(pocket: model.Pocket, table: Optional[InteractionTable], device: int) -> DevicePocket:
    from .docking import _pockets
    return _pockets.get(_ctx(device), pocket, table)


def grid_score(pose_coords: Coords, pocket: model.Pocket, device: int = 0) -> Union[int, np.ndarray]:
    """sum over atoms of the nearest grid node's value, -100 per atom outside."""
    P, single = _poses(pose_coords)
    out = np.zeros(P.shape[0], np.int32)
    check(lib().ds_op_grid_score(_ctx(device).handle, _device_pocket(pocket, None, device).handle, _p(P), P.shape[1],
                                 P.shape[0], _p(out)))
    return int(out[0]) if single else out


def bump_check(pose_coords: Coords, frag: model.Fragment, bump_distance: float = 0.8, early_exit: bool = True,
               counters: Optional[model.Counters] = None, device: int = 0):
    """any moving atom closer than bump_distance to a non-moving, non-axis atom.
    counters.bump_checks += pair evaluations of the sequential scan; bump_early_exits += 1 per pose
    whose scan stopped early."""
    P, single = _poses(pose_coords)
    bump = np.zeros(P.shape[0], np.uint8)
    pairs = np.zeros(P.shape[0], np.int64)
    check(lib().ds_op_bump_check(_ctx(device).handle, _p(P), P.shape[1], P.shape[0], int(frag.axis_begin),
                                 int(frag.axis_end), _p(_mask(frag)), float(bump_distance), int(bool(early_exit)),
                                 _p(bump), _p(pairs)))
    if counters is not None:
        counters.bump_checks += int(pairs.sum())
        if early_exit:
            counters.bump_early_exits += int(bump.astype(np.int64).sum())
    return bool(bump[0]) if single else bump.astype(bool)


def rescore(pose_coords: Coords, ligand_types, pocket: model.Pocket, table: Optional[InteractionTable] = None,
            cutoff: float = 8.0, device: int = 0):
    """sum over (ligand atom, pocket atom) pairs within the cutoff of table weight x bin
    multiplier, exact in fixed point 2^-24 (P11); returns the real value (chem_fx * 2^-24).
    ligand_types: a Ligand or the per-atom element codes."""
    P, single = _poses(pose_coords)
    types = ligand_types.types() if isinstance(ligand_types, model.Ligand) else np.asarray(ligand_types, np.uint8)
    types = np.ascontiguousarray(types, np.uint8)
    out = np.zeros(P.shape[0], np.int64)
    check(lib().ds_op_rescore(_ctx(device).handle, _device_pocket(pocket, table, device).handle, _p(P), _p(types),
                              P.shape[1], P.shape[0], C.c_float(cutoff), _p(out)))
    return float(out[0]) / CHEM_SCALE if single else out.astype(np.float64) / CHEM_SCALE


def rescore_fx(pose_coords: Coords, ligand_types, pocket: model.Pocket, table: Optional[InteractionTable] = None,
               cutoff: float = 8.0, device: int = 0) -> np.ndarray:
    """The fixed-point values themselves (int64, 2^-24) for every pose."""
    P, _ = _poses(pose_coords)
    types = ligand_types.types() if isinstance(ligand_types, model.Ligand) else np.asarray(ligand_types, np.uint8)
    types = np.ascontiguousarray(types, np.uint8)
    out = np.zeros(P.shape[0], np.int64)
    check(lib().ds_op_rescore(_ctx(device).handle, _device_pocket(pocket, table, device).handle, _p(P), _p(types),
                              P.shape[1], P.shape[0], C.c_float(cutoff), _p(out)))
    return out
