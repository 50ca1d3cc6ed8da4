"""Engines on the device: SPEC acceptance criterion 1 (engine equivalence over >= 1000 ligands
spanning all five atom ranges, workers in {1, 8}), the latency engine's allocate-once workspace
(SPEC.md:399), dock_ligand, and the batched engine's fill-ratio signal."""
import numpy as np
import pytest

import oracle
from paper_2209_05069_b200 import docking, engines, io, model
from paper_2209_05069_b200.bucketizer import classify
from paper_2209_05069_b200.native import InteractionTable, LigandBatch

pytestmark = pytest.mark.gpu


def _key(r):
    p = r.best_pose
    return (r.ligand_id, p.geometric_score, p.chem_fx, p.restart_index, p.align_indices, p.torsion_indices,
            p.coordinates.tobytes(), r.counters.poses_scored, r.counters.bump_checks, r.counters.bump_early_exits)


@pytest.fixture(scope="module")
def stream():
    b = io.generate_mixed_batch(1000, seed=14, heavy_range=(4, 80))
    ligs = b.to_ligands()
    assert {classify(l).atom_range_index for l in ligs} == {0, 1, 2, 3, 4}
    return b, ligs


def test_engine_equivalence_all_ranges(stream, synth_pocket, table):
    b, ligs = stream
    cfg = model.DockConfig()
    lat1 = engines.latency_engine.run(ligs, synth_pocket, cfg, workers=1, table=table)
    lat8 = engines.latency_engine.run(ligs, synth_pocket, cfg, workers=8, table=table)
    bat = engines.batched_engine.run(ligs, synth_pocket, cfg, workers=8, table=table)
    k1, k8, kb = ([_key(r) for r in rep.results] for rep in (lat1, lat8, bat))
    assert k1 == k8 == kb                                   # bit-identical, ordered by input sequence
    assert [e[:2] for e in lat1.errors] == [e[:2] for e in bat.errors]
    assert lat1.counters.poses_scored == bat.counters.poses_scored   # counter conservation
    assert lat8.workspace_allocations == 8 and lat8.extra_allocations == 0
    # and equal to the oracle on a subset spanning the ranges
    sub = list(range(0, 1000, 10))
    ob = b.subset(sub)
    o = oracle.dock_batch(ob, synth_pocket, table, cfg)
    byid = {r.ligand_id: r for r in lat1.results}
    for k, i in enumerate(sub):
        r = byid.get(b.ids[i])
        if o.results[k]["status"] != 0:
            assert r is None
            continue
        assert r.best_pose.geometric_score == o.results[k]["geom_score"]
        assert r.best_pose.chem_fx == o.results[k]["chem_fx"]
        assert r.best_pose.restart_index == o.results[k]["best_restart"]


def test_dock_ligand_and_errors(synth_pocket, table):
    lig = io.generate_dataset(20, 1, 1, seed=7)[0]
    r = docking.dock_ligand(lig, synth_pocket, model.DockConfig(), seed=0, table=table)
    o = oracle.dock_batch(LigandBatch.from_ligands([lig]), synth_pocket, table, model.DockConfig())
    assert r.best_pose.geometric_score == o.results[0]["geom_score"]
    assert abs(r.best_pose.chemical_score - o.results[0]["chem_fx"] / 2 ** 24) == 0
    assert np.array_equal(r.best_pose.coordinates, o.best_coords)
    bad = model.Ligand("bad", tuple(model.Atom.of(i, 0, 0, 1) for i in range(161)))
    with pytest.raises(model.TooManyAtoms):
        docking.dock_ligand(bad, synth_pocket)


def test_batched_engine_fill_ratio(synth_pocket, table):
    ligs = io.generate_dataset(10, 1, 10, seed=3)                   # 10 small ligands, capacity 1920
    rep = engines.batched_engine.run(ligs, synth_pocket, model.DockConfig(), workers=4, table=table)
    assert rep.counters.batches_dispatched == 1
    assert abs(rep.counters.batch_fill_ratio_sum - 10 / 1920) < 1e-12
    assert len(rep.results) + len(rep.errors) == 10
