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


def test_batched_engine_ligandbatch_fast_path_equals_ds_dock(synth_pocket, table):
    """batched_engine.run on a LigandBatch stream (zero-object path: native pack per producer chunk,
    bulk bucket push, dispatchers cutting batches out of the packed stream) gives ds_dock's records,
    best poses and torsions for every ligand, with SPEC, small and device capacities."""
    from paper_2209_05069_b200 import native
    from paper_2209_05069_b200.native import FAMILY_BATCHED, pack
    b = io.generate_mixed_batch(6000, seed=21)
    cfg = model.DockConfig()
    ref = docking.dock_batch(b, synth_pocket, cfg, seed=2, table=table)
    for caps, workers in ((None, 1), ({0: 333, 1: 257, 2: 100, 3: 64, 4: 32}, 4), ("device", 3)):
        rep = engines.batched_engine.run(b, synth_pocket, cfg, workers=workers, seed=2, table=table,
                                         capacities=caps, chunk=1000)
        rec = rep.records
        assert np.array_equal(rec["results"], ref.results), caps
        assert np.array_equal(rec["best_coords"][:len(ref.best_coords)], ref.best_coords)
        assert np.array_equal(rec["best_torsion"][:len(ref.best_torsion)], ref.best_torsion)
        assert len(rep.results) + len(rep.errors) == b.n
        assert sum(e["size"] for e in rep.dispatch_log) == b.n
        assert rep.counters.batches_dispatched == len(rep.dispatch_log)


def test_batched_engine_dispatch_log_monotone(synth_pocket, table):
    """the batched engine never begins a batch before it is full or flushed — per
    bucket the dispatch log is monotone (detach <= start, full batches of exactly capacity before
    the flushed partial), and the observed counters match the log."""
    b = io.generate_mixed_batch(5000, seed=22)
    caps = {0: 97, 1: 61, 2: 43, 3: 29, 4: 13}
    rep = engines.batched_engine.run(b, synth_pocket, model.DockConfig(), workers=4, table=table, capacities=caps,
                                     chunk=700)
    per = {}
    for e in rep.dispatch_log:
        assert e["started"] >= e["detached"] and e["finished"] >= e["started"]
        per.setdefault(e["key"], []).append(e)
    for key, es in per.items():
        es.sort(key=lambda e: e["detached"])
        kinds = [e["kind"] for e in es]
        assert kinds.count("flush") <= 1 and (kinds[-1] == "flush" or "flush" not in kinds)
        assert all(e["size"] == caps[key[0]] for e in es if e["kind"] == "full")
        assert all(0 < e["size"] <= caps[key[0]] for e in es)
    fill = sum(e["size"] / e["capacity"] for e in rep.dispatch_log)
    assert abs(rep.counters.batch_fill_ratio_sum - fill) < 1e-9
    assert rep.counters.batches_dispatched == len(rep.dispatch_log)


def test_batched_engine_homogeneous_capacity_example(synth_pocket, table):
    """a homogeneous stream of 3840 small ligands -> 2 full batches, fill ratio 1.0."""
    b = io.generate_dataset_batch(10, 1, 3840, seed=5)
    rep = engines.batched_engine.run(b, synth_pocket, model.DockConfig(), workers=2, table=table)
    assert rep.counters.batches_dispatched == 2
    assert rep.counters.batch_fill_ratio_sum == 2.0
    assert all(e["kind"] == "full" and e["size"] == 1920 for e in rep.dispatch_log)


def test_device_capacities_from_occupancy(gpu_ctx):
    """ds_query_capacity: occupancy-derived, identical for every range (the kernels are not
    range-specialised), a multiple of the SM count."""
    import torch
    from paper_2209_05069_b200.bucketizer import device_capacities
    caps = device_capacities(gpu_ctx)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    assert set(caps) == {0, 1, 2, 3, 4} and len(set(caps.values())) == 1
    c = caps[0]
    assert c > 0 and c % sms == 0 and c >= sms * 8


def test_engines_record_invalid_ligands_and_continue(synth_pocket, table):
    """Per-ligand validation errors are recorded with their input sequence and the stream continues
    (SPEC.md:395, 405); both engines agree."""
    ligs = io.generate_dataset(12, 2, 6, seed=8)
    bad = model.Ligand("too_many", tuple(model.Atom.of(i, 0, 0, 1) for i in range(161)))
    stream = ligs[:2] + [bad] + ligs[2:]
    for run in (engines.batched_engine.run, engines.latency_engine.run):
        rep = run(stream, synth_pocket, model.DockConfig(), workers=2, table=table)
        assert [e[:2] for e in rep.errors] == [(2, "too_many")]
        assert [r.ligand_id for r in rep.results] == [l.id for l in ligs]


def test_engine_fatal_config_error_raises(synth_pocket, table):
    """A configuration the device rejects (alignment_step_deg=1: 360^2 rotations exceed the 16-bit
    argmax key) is fatal: run() raises instead of returning a short report."""
    from paper_2209_05069_b200.native import DsError
    ligs = io.generate_dataset(12, 2, 3, seed=8)
    cfg = model.DockConfig(alignment_step_deg=1)
    for run in (engines.batched_engine.run, engines.latency_engine.run):
        with pytest.raises(DsError):
            run(ligs, synth_pocket, cfg, workers=2, table=table)


def test_engine_stream_index_lists_equal_ds_dock(synth_pocket, table):
    """ds_stream (the batched engine's device-resident stream): the ligands docked as shuffled index
    lists on two contexts, uploaded in ranges, give ds_dock's records, poses and torsions; ligands no
    list names read back as zero records; a config with other restarts is refused."""
    from paper_2209_05069_b200.native import Context, EngineStream, RESULT_DTYPE, pack, pinned_copy
    b = io.generate_mixed_batch(3000, seed=23)
    cfg = model.DockConfig()
    p = pack(b)
    ctx0, ctx1 = Context(0), Context(0)
    ref = ctx0.dock(ctx0.pocket(synth_pocket, table), p, cfg, seed=4)
    es = EngineStream(ctx0)
    es.begin(p.atom_off, p.frag_off, cfg.restarts_n)
    xyzt, fdesc, idh = pinned_copy(p.atom_xyzt), pinned_copy(p.frag_desc), pinned_copy(p.id_hash)
    for lo in range(0, b.n, 700):
        es.upload(lo, min(b.n, lo + 700), xyzt, fdesc, idh)
    perm = np.random.default_rng(0).permutation(b.n - 10).astype(np.int32)   # the last 10: never docked
    es.dock(ctx0, ctx0.pocket(synth_pocket, table), perm[:1234], cfg, seed=4)
    es.dock(ctx1, ctx1.pocket(synth_pocket, table), perm[1234:], cfg, seed=4)
    res = np.empty(b.n, RESULT_DTYPE)
    co = np.empty((int(p.atom_off[-1]), 3), np.float32)
    to = np.empty(int(p.frag_off[-1]), np.uint8)
    es.download(ctx0, res, co, to)
    n = b.n - 10
    assert np.array_equal(res[:n], ref.results[:n])
    a_n, f_n = int(p.atom_off[n]), int(p.frag_off[n])
    assert np.array_equal(co[:a_n], ref.best_coords[:a_n]) and np.array_equal(to[:f_n], ref.best_torsion[:f_n])
    assert not res[n:].view(np.uint8).any()
    with pytest.raises(ValueError):   # DS_ERR_INVALID_ARG
        es.dock(ctx0, ctx0.pocket(synth_pocket, table), perm[:5], model.DockConfig(restarts_n=4), seed=4)
    es.close()


def test_batched_engine_concurrent_runs(synth_pocket, table):
    """Two batched_engine.run calls at once (each takes its own device stream and arena from the
    pools) give the same results as one at a time."""
    import threading
    b1, b2 = io.generate_mixed_batch(2500, seed=24), io.generate_mixed_batch(1800, seed=25)
    cfg = model.DockConfig()
    solo = [engines.batched_engine.run(b, synth_pocket, cfg, table=table).records["results"] for b in (b1, b2)]
    out = [None, None]

    def go(k, b):
        out[k] = engines.batched_engine.run(b, synth_pocket, cfg, table=table, capacities={0: 200, 1: 150, 2: 100,
                                                                                          3: 50, 4: 20})
    ts = [threading.Thread(target=go, args=(k, b)) for k, b in enumerate((b1, b2))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for k in range(2):
        assert np.array_equal(out[k].records["results"], solo[k])


def test_batched_engine_nondefault_config_equals_ds_dock(synth_pocket, table):
    """The engine stream with another restart count, top-K, angle steps and no early exit: the
    records, poses and torsions equal one ds_dock of the whole batch."""
    from paper_2209_05069_b200.native import Context, pack
    b = io.generate_mixed_batch(2500, seed=26)
    cfg = model.DockConfig(restarts_n=12, rescore_top_k=6, alignment_step_deg=10, torsion_step_deg=30,
                           early_exit=False)
    ctx = Context(0)
    ref = ctx.dock(ctx.pocket(synth_pocket, table), pack(b), cfg, seed=3)
    rep = engines.batched_engine.run(b, synth_pocket, cfg, seed=3, table=table, workers=3,
                                     capacities={0: 300, 1: 200, 2: 100, 3: 60, 4: 20}, chunk=400)
    rec = rep.records
    assert np.array_equal(rec["results"], ref.results)
    assert np.array_equal(rec["best_coords"][:len(ref.best_coords)], ref.best_coords)
    assert np.array_equal(rec["best_torsion"][:len(ref.best_torsion)], ref.best_torsion)
