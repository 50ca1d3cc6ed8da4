"""docking: Alg. 1 for one ligand, executed on the B200.

`dock_ligand` keeps the reference signature.  The whole pipeline — starting
poses, the n_a^2 rigid sweep, the greedy torsion sweep with bump checks, select_poses and
rescoring — runs in libdockscreen's sm_100a kernels; this module only packs inputs and maps
the result records back to DockResult.
"""
from __future__ import annotations

import threading
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import model
from .native import (CHEM_SCALE, FAMILY_BATCHED, FAMILY_LATENCY, STATUS_DEGENERATE_AXIS, STATUS_NO_VALID_POSE,
                     Context, DevicePocket, DockOutput, InteractionTable, LigandBatch, PackedBatch, pack)

_tls = threading.local()


def thread_context(device: int = 0) -> Context:
    """One ds_ctx per host thread and device."""
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if device not in ctxs:
        ctxs[device] = Context(device)
    return ctxs[device]


class PocketCache:
    """Device copies of a pocket, cached on the context that owns them (read-only, shared by all
    of that context's calls); they are released with the context."""

    def get(self, ctx: Context, pocket: model.Pocket, table: Optional[InteractionTable]) -> DevicePocket:
        cache = ctx.__dict__.setdefault("_pocket_cache", {})
        key = (id(pocket), id(table))
        hit = cache.get(key)
        if hit is None or hit[0] is not pocket or hit[1] is not table:
            hit = (pocket, table, ctx.pocket(pocket, table))
            cache[key] = hit
        return hit[2]


_pockets = PocketCache()


def results_from_output(batch: LigandBatch, out: DockOutput, cfg: model.DockConfig) -> List[model.DockResult]:
    """Map ds_result records (+ best coordinates / torsions) to SPEC DockResults."""
    res = out.results
    results: List[model.DockResult] = []
    for i in range(batch.n):
        r = res[i]
        c = model.Counters(poses_scored=int(r["poses_scored"]), bump_checks=int(r["bump_checks"]),
                           bump_early_exits=int(r["bump_early_exits"]))
        st = int(r["status"])
        if st == STATUS_NO_VALID_POSE:
            results.append(model.DockResult(batch.ids[i], None, c, "no valid pose"))
            continue
        if st == STATUS_DEGENERATE_AXIS:
            results.append(model.DockResult(batch.ids[i], None, c, "DegenerateAxis"))
            continue
        if st != 0:
            results.append(model.DockResult(batch.ids[i], None, c, f"status {st}"))
            continue
        a0, a1 = int(batch.atom_off[i]), int(batch.atom_off[i + 1])
        f0, f1 = int(batch.frag_off[i]), int(batch.frag_off[i + 1])
        coords = out.best_coords[a0:a1].copy() if out.best_coords is not None else None
        pose = model.Pose(coordinates=coords, geometric_score=int(r["geom_score"]),
                          chemical_score=float(r["chem_fx"]) / CHEM_SCALE, restart_index=int(r["best_restart"]),
                          valid=True, align_indices=(int(r["best_ax"]), int(r["best_ay"])),
                          torsion_indices=tuple(int(t) for t in out.best_torsion[f0:f1]), chem_fx=int(r["chem_fx"]))
        results.append(model.DockResult(batch.ids[i], pose, c))
    return results


def dock_batch(batch: LigandBatch, pocket: model.Pocket, cfg: model.DockConfig = model.DockConfig(), seed: int = 0,
               table: Optional[InteractionTable] = None, family: int = FAMILY_BATCHED, device: int = 0,
               packed: Optional[PackedBatch] = None, detail: bool = False) -> DockOutput:
    ctx = thread_context(device)
    dp = _pockets.get(ctx, pocket, table)
    return ctx.dock(dp, packed if packed is not None else pack(batch), cfg, seed, family, coords=True, detail=detail)


def dock_ligand(ligand: model.Ligand, pocket: model.Pocket, cfg: model.DockConfig = model.DockConfig(), seed: int = 0,
                table: Optional[InteractionTable] = None, family: int = FAMILY_LATENCY,
                device: int = 0) -> model.DockResult:
    """SPEC.md:277.  Raises NoValidPose / DegenerateAxis like the reference."""
    model.validate_ligand(ligand)
    batch = LigandBatch.from_ligands([ligand])
    out = dock_batch(batch, pocket, cfg, seed, table, family, device)
    r = results_from_output(batch, out, cfg)[0]
    if r.error == "no valid pose":
        raise model.NoValidPose(ligand.id)
    if r.error == "DegenerateAxis":
        raise model.DegenerateAxis(ligand.id)
    return r
