"""GPU parity: the sm_100a kernels against the CPU oracle, bit-exact."""
import numpy as np
import pytest

import oracle
from helpers import compare
from paper_2209_05069_b200 import io, model, native
from paper_2209_05069_b200.native import FAMILY_BATCHED, FAMILY_LATENCY, pack

pytestmark = pytest.mark.gpu


def _run(ctx, batch, pocket, table, cfg, seed=0, family=FAMILY_BATCHED):
    dp = ctx.pocket(pocket, table)
    g = ctx.dock(dp, pack(batch), cfg, seed, family, coords=True, detail=True)
    o = oracle.dock_batch(batch, pocket, table, cfg, seed)
    return g, o


@pytest.mark.parametrize("shape", [(12, 5), (20, 1), (6, 0), (30, 12)])
def test_batched_parity_shapes(gpu_ctx, synth_pocket, table, shape):
    batch = io.generate_dataset_batch(shape[0], shape[1], 48, seed=1)
    cfg = model.DockConfig()
    g, o = _run(gpu_ctx, batch, synth_pocket, table, cfg)
    compare(batch, g, o, cfg)


def test_batched_parity_mixed(gpu_ctx, synth_pocket, table):
    batch = io.generate_mixed_batch(200, seed=3)
    cfg = model.DockConfig()
    g, o = _run(gpu_ctx, batch, synth_pocket, table, cfg)
    compare(batch, g, o, cfg)


@pytest.mark.parametrize("shape", [(12, 5), (36, 20), (8, 0)])
def test_latency_parity_shapes(gpu_ctx, synth_pocket, table, shape):
    """Latency family (one ligand spread over the GPU) against the oracle, one ligand per call and
    a small batch per call."""
    cfg = model.DockConfig()
    batch = io.generate_dataset_batch(shape[0], shape[1], 6, seed=2)
    for i in range(2):
        one = batch.subset([i])
        g, o = _run(gpu_ctx, one, synth_pocket, table, cfg, family=FAMILY_LATENCY)
        compare(one, g, o, cfg)
    g, o = _run(gpu_ctx, batch, synth_pocket, table, cfg, family=FAMILY_LATENCY)
    compare(batch, g, o, cfg)


def test_latency_parity_mixed_and_options(gpu_ctx, synth_pocket, table):
    batch = io.generate_mixed_batch(40, seed=6)
    for cfg in (model.DockConfig(), model.DockConfig(early_exit=False),
                model.DockConfig(restarts_n=5, rescore_top_k=3, alignment_step_deg=20, torsion_step_deg=30)):
        g, o = _run(gpu_ctx, batch, synth_pocket, table, cfg, family=FAMILY_LATENCY)
        compare(batch, g, o, cfg)
        if not cfg.early_exit:
            assert np.array_equal(g.results["bump_checks"].astype(np.int64), o.results["bump_checks"])


@pytest.mark.parametrize("restarts", [1, 12, 32])
def test_latency_cluster_alignment_restart_counts(gpu_ctx, synth_pocket, table, restarts):
    """The latency alignment for the default 12-degree step is one 8-CTA cluster per (ligand,
    restart) with a DSMEM reduction to the argmax key: grids of L x N clusters for N = 1 .. 32,
    ligands from 3 to 160 atoms (fewer atoms than the cluster's 32 warps included)."""
    batch = io.generate_mixed_batch(12, seed=13)
    small = io.generate_dataset_batch(1, 0, 2, seed=3)     # 2-3 atoms
    big = io.generate_dataset_batch(70, 30, 2, seed=4)     # 160 atoms
    cfg = model.DockConfig(restarts_n=restarts, rescore_top_k=min(4, restarts))
    for b in (batch, small, big):
        g, o = _run(gpu_ctx, b, synth_pocket, table, cfg, seed=5, family=FAMILY_LATENCY)
        compare(b, g, o, cfg)


def test_families_agree(gpu_ctx, synth_pocket, table):
    """Engine equivalence on the device: both families, identical records."""
    batch = io.generate_mixed_batch(100, seed=8)
    cfg = model.DockConfig()
    dp = gpu_ctx.pocket(synth_pocket, table)
    a = gpu_ctx.dock(dp, pack(batch), cfg, 3, FAMILY_BATCHED, coords=True, detail=True)
    b = gpu_ctx.dock(dp, pack(batch), cfg, 3, FAMILY_LATENCY, coords=True, detail=True)
    for f in ("status", "geom_score", "chem_fx", "best_restart", "best_ax", "best_ay", "n_kept", "poses_scored",
              "bump_early_exits"):
        assert np.array_equal(a.results[f], b.results[f]), f
    assert np.array_equal(a.best_coords, b.best_coords)
    assert np.array_equal(a.restart_torsion, b.restart_torsion)


def test_batched_options(gpu_ctx, synth_pocket, table):
    """Non-default DockConfig on the batched family (generic alignment kernel path)."""
    batch = io.generate_mixed_batch(60, seed=9)
    for cfg in (model.DockConfig(restarts_n=5, rescore_top_k=3, alignment_step_deg=20, torsion_step_deg=30),
                model.DockConfig(restarts_n=12, rescore_top_k=6, alignment_step_deg=10, similarity_rmsd=0.5)):
        g, o = _run(gpu_ctx, batch, synth_pocket, table, cfg, seed=4)
        compare(batch, g, o, cfg)


def test_l2_variant_pocket_global_grid(gpu_ctx, table):
    """Spacing 0.375 Å (75^3-class grid, too large for shared memory): the LDG/L2 path."""
    pocket = io.synthetic_pocket(spacing=0.375)
    batch = io.generate_mixed_batch(60, seed=10)
    cfg = model.DockConfig()
    g, o = _run(gpu_ctx, batch, pocket, table, cfg)
    compare(batch, g, o, cfg)


def test_pipelined_ds_dock_matches_resident(gpu_ctx, synth_pocket, table):
    """ds_dock on a large batch (chunked H2D/compute/D2H pipeline) == the resident single-launch
    path, record for record; and a spread subset == the oracle."""
    from paper_2209_05069_b200.native import ResidentBatch
    batch = io.generate_mixed_batch(24000, seed=17)
    cfg = model.DockConfig()
    dp = gpu_ctx.pocket(synth_pocket, table)
    packed = pack(batch)
    g = gpu_ctx.dock(dp, packed, cfg, 2, FAMILY_BATCHED, coords=True, detail=True)
    rb = ResidentBatch(gpu_ctx, packed)
    rb.dock(dp, cfg, seed=2)
    r = rb.download()
    assert np.array_equal(g.results, r)
    sub = list(range(0, 24000, 97))
    sb = batch.subset(sub)
    o = oracle.dock_batch(sb, synth_pocket, table, cfg, 2)
    for f in ("status", "geom_score", "chem_fx", "best_restart", "best_ax", "best_ay", "n_kept", "poses_scored"):
        assert np.array_equal(g.results[f][sub].astype(np.int64), o.results[f].astype(np.int64)), f
    for k, i in enumerate(sub):
        a0, a1 = batch.atom_off[i], batch.atom_off[i + 1]
        b0, b1 = sb.atom_off[k], sb.atom_off[k + 1]
        if o.results[k]["status"] == 0:
            assert np.array_equal(g.best_coords[a0:a1], o.best_coords[b0:b1])


def test_batched_parity_no_early_exit(gpu_ctx, synth_pocket, table):
    batch = io.generate_mixed_batch(64, seed=4)
    cfg = model.DockConfig(early_exit=False)
    g, o = _run(gpu_ctx, batch, synth_pocket, table, cfg)
    compare(batch, g, o, cfg)
    assert np.array_equal(g.results["bump_checks"].astype(np.int64), o.results["bump_checks"])


def _scaled(batch, scale):
    """The same ligands with every coordinate scaled (crowded when scale < 1: bonds of 1.5*scale Å)."""
    from paper_2209_05069_b200.native import LigandBatch
    return LigandBatch(batch.atom_off, (batch.atom_xyz * np.float32(scale)).astype(np.float32), batch.atom_type,
                       batch.bond_off, batch.bonds, batch.frag_off, batch.frag_axis, batch.frag_mask, batch.ids)


@pytest.mark.parametrize("scale", [0.7, 0.45])
def test_batched_parity_crowded(gpu_ctx, synth_pocket, table, scale):
    """Crowded ligands: many bump candidates per moving atom, so the inline slots, the per-fragment
    overflow list and its full-scan fallback (> 32 overflow pairs) all run; both early-exit modes."""
    batch = _scaled(io.generate_dataset_batch(36, 20, 40, seed=4), scale)
    for cfg in (model.DockConfig(), model.DockConfig(early_exit=False)):
        g, o = _run(gpu_ctx, batch, synth_pocket, table, cfg)
        compare(batch, g, o, cfg)


def test_batched_parity_fine_torsion_step(gpu_ctx, synth_pocket, table):
    """torsion_step_deg = 10: 36 angles, so the sweep runs a second angle block (device-computed
    lane layout in the batched family, a second CTA block pass in the latency family)."""
    batch = io.generate_mixed_batch(60, seed=6)
    cfg = model.DockConfig(torsion_step_deg=10)
    for fam in (FAMILY_BATCHED, FAMILY_LATENCY):
        g, o = _run(gpu_ctx, batch, synth_pocket, table, cfg, family=fam)
        compare(batch, g, o, cfg)


@pytest.mark.parametrize("spacing,padding,natoms", [(0.5, 4.0, 200), (0.375, 4.0, 200), (0.8, 2.0, 30), (1.0, 4.0, 1)])
def test_build_pocket_device_matches_host(gpu_ctx, spacing, padding, natoms):
    """the GPU build_pocket grid is bit-identical to the host build (P18)."""
    atoms = io.pocket_atoms(natoms, seed=7) if natoms > 1 else [model.Atom.of(0.0, 0.0, 0.0, 3)]
    host = io.build_pocket(atoms, spacing, padding)
    dev = io.build_pocket(atoms, spacing, padding, ctx=gpu_ctx)
    assert dev.grid_origin == host.grid_origin and dev.grid_dims == host.grid_dims
    assert np.array_equal(np.asarray(dev.grid_values), np.asarray(host.grid_values))


@pytest.mark.parametrize("n", [64, 6000])
def test_ds_dock_transfer_paths_match_resident(gpu_ctx, synth_pocket, table, n):
    """Both unchunked ds_dock transfer paths — the express path (n = 64: one H2D of a packed input
    arena, one D2H of an output arena) and the per-array path (n = 6000: > 4 MB of inputs) — give
    the resident path's records, best poses and per-restart detail, for both kernel families."""
    from paper_2209_05069_b200.native import FAMILY_LATENCY, ResidentBatch
    batch = io.generate_mixed_batch(n, seed=23)
    cfg = model.DockConfig()
    dp = gpu_ctx.pocket(synth_pocket, table)
    packed = pack(batch)
    for fam in (FAMILY_BATCHED, FAMILY_LATENCY) if n <= 64 else (FAMILY_BATCHED,):
        g = gpu_ctx.dock(dp, packed, cfg, 1, fam, coords=True, detail=True)
        rb = ResidentBatch(gpu_ctx, packed)
        rb.dock(dp, cfg, seed=1, family=fam)
        r = rb.download()
        rb.close()
        # every field, counters included (bump_checks is the sequential scan's exact count, P14)
        for f in r.dtype.names:
            assert np.array_equal(g.results[f], r[f]), (fam, f)
    if n <= 64:
        o = oracle.dock_batch(batch, synth_pocket, table, cfg, 1)
        compare(batch, g, o, cfg)


def test_parity_large_mixed_both_families(gpu_ctx, synth_pocket, table):
    """2,000 mixed config-3 ligands through the batched family and 300 through the latency family,
    every field against the oracle (rare paths: overflow lists, all-bump fragments, invalid poses)."""
    batch = io.generate_mixed_batch(2000, seed=31)
    cfg = model.DockConfig()
    g, o = _run(gpu_ctx, batch, synth_pocket, table, cfg, seed=5)
    compare(batch, g, o, cfg)
    sub = batch.subset(range(0, 2000, 7)[:300])
    g, o = _run(gpu_ctx, sub, synth_pocket, table, cfg, seed=5, family=FAMILY_LATENCY)
    compare(sub, g, o, cfg)


def test_parity_maximum_ligands(gpu_ctx, synth_pocket, table):
    """DS_MAX_ATOMS (160-atom) ligands with 60 rotatable bonds: five 32-atom slots, up to 158 moving
    atoms per fragment, the largest per-warp records — both families against the oracle."""
    batch = io.generate_dataset_batch(70, 60, 6, seed=9)
    assert int(np.diff(batch.atom_off).max()) == 160
    cfg = model.DockConfig()
    for fam in (FAMILY_BATCHED, FAMILY_LATENCY):
        g, o = _run(gpu_ctx, batch, synth_pocket, table, cfg, seed=2, family=fam)
        compare(batch, g, o, cfg)


def test_parity_large_weights_no_int32_overflow(gpu_ctx, synth_pocket):
    """Bin multipliers near the fixed-point limit (|W| ~ 2^30): the rescore's int32 partial sums
    must be sized so they cannot overflow (PocketView::part_terms) — both families vs the oracle."""
    from paper_2209_05069_b200.native import InteractionTable
    base = InteractionTable.default()
    table = InteractionTable(np.clip(base.table * 1.0, -1, 1), ((2.0, 100.0), (4.0, 64.0), (6.0, 32.0), (8.0, 16.0)))
    batch = io.generate_mixed_batch(48, seed=41)
    cfg = model.DockConfig()
    for fam in (FAMILY_BATCHED, FAMILY_LATENCY):
        g, o = _run(gpu_ctx, batch, synth_pocket, table, cfg, seed=1, family=fam)
        compare(batch, g, o, cfg)


def test_degenerate_axis_both_families(gpu_ctx, synth_pocket, table):
    """DegenerateAxis: a fragment whose two axis atoms coincide stops the ligand
    with status DEGENERATE_AXIS in both families, as in the oracle; the other ligands of the batch
    are unaffected."""
    batch = io.generate_dataset_batch(20, 6, 8, seed=21)
    xyz = batch.atom_xyz.copy()
    for i in (1, 4, 6):  # ligands with a degenerate fragment (fragment i % 3 of the ligand)
        a0, f0 = int(batch.atom_off[i]), int(batch.frag_off[i])
        b, e = batch.frag_axis[f0 + i % 3]
        xyz[a0 + e] = xyz[a0 + b]
    bad = native.LigandBatch(batch.atom_off, xyz, batch.atom_type, batch.bond_off, batch.bonds, batch.frag_off,
                             batch.frag_axis, batch.frag_mask, list(batch.ids))
    cfg = model.DockConfig()
    for fam in (FAMILY_BATCHED, FAMILY_LATENCY):
        g, o = _run(gpu_ctx, bad, synth_pocket, table, cfg, seed=1, family=fam)
        assert (o.results["status"][[1, 4, 6]] == native.STATUS_DEGENERATE_AXIS).all()
        compare(bad, g, o, cfg)


@pytest.mark.parametrize("rmsd,k", [(4.0, 4), (15.0, 8), (40.0, 3), (15.0, 1)])
def test_select_exact_rmsd_path(gpu_ctx, synth_pocket, table, rmsd, k):
    """Large similarity thresholds: the centroid bound rarely separates poses, so most pairs take
    the exact sequential RMSD (the kept pose replayed into the second slot) and many candidates are
    rejected — both families against the oracle, every field."""
    batch = io.generate_mixed_batch(80, seed=31)
    cfg = model.DockConfig(restarts_n=8, rescore_top_k=k, similarity_rmsd=rmsd)
    for fam in (FAMILY_BATCHED, FAMILY_LATENCY):
        g, o = _run(gpu_ctx, batch, synth_pocket, table, cfg, seed=7, family=fam)
        compare(batch, g, o, cfg)
    kept = o.results["n_kept"][o.results["status"] == 0]
    if rmsd >= 15.0 and k > 1:
        assert (kept < k).any()   # the threshold rejects candidates: the exact path decided some
