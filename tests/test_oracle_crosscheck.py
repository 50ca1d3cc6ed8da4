"""Pin the C oracle with a second, independent restatement (oracle/pyoracle.py, exact f32
emulation in pure Python): both must agree bit for bit on every selected index and score."""
import numpy as np
import pytest

import oracle
import pyoracle as py
from paper_2209_05069_b200 import io, model
from paper_2209_05069_b200.native import InteractionTable


def _py_pocket(pocket, table):
    xyz, typ = pocket.atom_arrays()
    return py.Pocket(pocket.grid_origin, pocket.grid_spacing, pocket.grid_dims, pocket.grid_values, xyz, typ,
                     table.table, table.bins)


def _py_ligand(batch, i):
    a0, a1 = batch.atom_off[i], batch.atom_off[i + 1]
    f0, f1 = batch.frag_off[i], batch.frag_off[i + 1]
    masks = []
    for f in range(f0, f1):
        bits = batch.frag_mask[f]
        masks.append({k for k in range(a1 - a0) if (int(bits[k >> 5]) >> (k & 31)) & 1})
    return py.Ligand(batch.ids[i], batch.atom_xyz[a0:a1], batch.atom_type[a0:a1],
                     [tuple(x) for x in batch.frag_axis[f0:f1]], masks)


def _check(batch, pocket, table, cfg, seed=0):
    orc = oracle.dock_batch(batch, pocket, table, cfg, seed)
    P = _py_pocket(pocket, table)
    for i in range(batch.n):
        ref = py.dock_ligand(_py_ligand(batch, i), P, cfg, seed)
        r = orc.results[i]
        assert r["status"] == ref["status"]
        if ref["status"] != 0:
            continue
        assert r["geom_score"] == ref["geom"] and r["chem_fx"] == ref["chem_fx"]
        assert r["best_restart"] == ref["best_restart"]
        rr = orc.restarts[i]
        for k, (ix, iy, sc) in enumerate(ref["aligns"]):
            assert (rr[k]["ax"], rr[k]["ay"], rr[k]["align_score"]) == (ix, iy, sc)
            assert rr[k]["final_geom"] == ref["final_geom"][k] and bool(rr[k]["valid"]) == ref["valid"][k]
        f0, f1 = batch.frag_off[i], batch.frag_off[i + 1]
        for k in range(cfg.restarts_n):
            assert list(orc.restart_torsion[f0:f1, k]) == ref["tors"][k]
        kept = sorted([k for k in range(cfg.restarts_n) if rr[k]["kept"]], key=lambda k: rr[k]["kept"])
        assert kept == ref["kept"]


@pytest.mark.parametrize("heavy,frags", [(4, 1), (5, 2), (6, 3)])
def test_crosscheck_coarse_angles(heavy, frags):
    """Small chain ligands, coarse alignment grid (36°: 100 rotations) to keep pure Python fast."""
    pocket = io.synthetic_pocket()
    table = InteractionTable.default()
    batch = io.generate_dataset_batch(heavy, frags, 3, seed=21)
    cfg = model.DockConfig(restarts_n=4, rescore_top_k=2, alignment_step_deg=36, torsion_step_deg=36)
    _check(batch, pocket, table, cfg)


def test_crosscheck_default_angles():
    """Default DockConfig angles (900 rotations, 10 torsion angles) on one tiny ligand."""
    pocket = io.synthetic_pocket()
    table = InteractionTable.default()
    batch = io.generate_dataset_batch(3, 1, 1, seed=22)
    cfg = model.DockConfig(restarts_n=2, rescore_top_k=2)
    _check(batch, pocket, table, cfg, seed=5)


def test_crosscheck_no_early_exit_and_fine_torsion():
    pocket = io.synthetic_pocket(spacing=0.375)
    table = InteractionTable.default()
    batch = io.generate_dataset_batch(5, 2, 2, seed=23)
    cfg = model.DockConfig(restarts_n=3, rescore_top_k=3, alignment_step_deg=60, torsion_step_deg=20,
                           early_exit=False)
    _check(batch, pocket, table, cfg, seed=7)
