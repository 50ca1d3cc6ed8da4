"""The latency family's cluster-speculative optimisation kernel: one (ligand,
restart) over a cluster of n_t CTAs that evaluates fragment pairs (a lead thread group sweeps f on
the current pose, a thread group of CTA h sweeps f + 1 under f's commit of angle h).  Its results must be bit-identical to the oracle and to
the sequential one-CTA fragment chain, for every shape the chain has: no fragments, one, odd and
even fragment counts, all-bumped fragments, degenerate axes at even and odd positions, early exit
off, maximum ligands, restart counts that run the clusters in several waves.

DS_LATENCY_SPEC forces the variant (1 = spread whenever it applies, 0 = never); unset, the
library spreads a call when all its clusters are resident at once (one ligand, N <= 8)."""
import numpy as np
import pytest

import oracle
from helpers import compare
from paper_2209_05069_b200 import io, model, native
from paper_2209_05069_b200.native import FAMILY_LATENCY, pack

pytestmark = pytest.mark.gpu


def _dock(ctx, dp, batch, cfg, seed):
    return ctx.dock(dp, pack(batch), cfg, seed, FAMILY_LATENCY, coords=True, detail=True)


def _both(monkeypatch, ctx, dp, batch, cfg, seed):
    monkeypatch.setenv("DS_LATENCY_SPEC", "1")
    s = _dock(ctx, dp, batch, cfg, seed)
    monkeypatch.setenv("DS_LATENCY_SPEC", "0")
    q = _dock(ctx, dp, batch, cfg, seed)
    monkeypatch.delenv("DS_LATENCY_SPEC")
    return s, q


def _same(s, q, batch):
    for f in s.results.dtype.names:
        assert np.array_equal(s.results[f], q.results[f]), f
    # best poses exist for OK ligands only (the others' output rows are not written)
    ok = s.results["status"] == native.STATUS_OK
    for i in np.nonzero(ok)[0]:
        a0, a1 = batch.atom_off[i], batch.atom_off[i + 1]
        f0, f1 = batch.frag_off[i], batch.frag_off[i + 1]
        assert np.array_equal(s.best_coords[a0:a1], q.best_coords[a0:a1])
        assert np.array_equal(s.best_torsion[f0:f1], q.best_torsion[f0:f1])
    for f in s.restarts.dtype.names:
        assert np.array_equal(s.restarts[f], q.restarts[f]), (f, s.restarts[f], q.restarts[f])
    assert np.array_equal(s.restart_torsion, q.restart_torsion)


@pytest.mark.parametrize("shape", [(8, 0), (12, 1), (12, 2), (12, 5), (30, 12), (36, 20), (36, 21)])
def test_spread_kernel_matches_oracle_and_chain(monkeypatch, gpu_ctx, synth_pocket, table, shape):
    cfg = model.DockConfig()
    dp = gpu_ctx.pocket(synth_pocket, table)
    batch = io.generate_dataset_batch(shape[0], shape[1], 4, seed=11)
    for i in range(2):
        one = batch.subset([i])
        s, q = _both(monkeypatch, gpu_ctx, dp, one, cfg, 3)
        assert s.stats.lat_spread == 10 and q.stats.lat_spread == 1
        _same(s, q, one)
        compare(one, s, oracle.dock_batch(one, synth_pocket, table, cfg, 3), cfg)
    s, q = _both(monkeypatch, gpu_ctx, dp, batch, cfg, 3)
    _same(s, q, batch)
    compare(batch, s, oracle.dock_batch(batch, synth_pocket, table, cfg, 3), cfg)


def test_spread_kernel_mixed_options_and_waves(monkeypatch, gpu_ctx, synth_pocket, table):
    """Mixed config-3 ligands (many all-bumped fragments), early exit off, and 12 / 32 restarts
    (clusters in several waves); a non-default torsion step falls back to the chain."""
    dp = gpu_ctx.pocket(synth_pocket, table)
    batch = io.generate_mixed_batch(24, seed=17)
    for cfg in (model.DockConfig(), model.DockConfig(early_exit=False),
                model.DockConfig(restarts_n=12, rescore_top_k=4), model.DockConfig(restarts_n=32, rescore_top_k=5)):
        s, q = _both(monkeypatch, gpu_ctx, dp, batch, cfg, 5)
        assert s.stats.lat_spread == 10
        _same(s, q, batch)
        compare(batch, s, oracle.dock_batch(batch, synth_pocket, table, cfg, 5), cfg)
    cfg = model.DockConfig(torsion_step_deg=30)
    two = batch.subset([0, 1])
    s, q = _both(monkeypatch, gpu_ctx, dp, two, cfg, 5)
    assert s.stats.lat_spread == 1
    _same(s, q, two)


def test_spread_kernel_maximum_ligands(monkeypatch, gpu_ctx, synth_pocket, table):
    batch = io.generate_dataset_batch(70, 60, 3, seed=9)
    cfg = model.DockConfig()
    dp = gpu_ctx.pocket(synth_pocket, table)
    s, q = _both(monkeypatch, gpu_ctx, dp, batch, cfg, 2)
    _same(s, q, batch)
    compare(batch, s, oracle.dock_batch(batch, synth_pocket, table, cfg, 2), cfg)


def test_spread_kernel_degenerate_axis_even_and_odd(monkeypatch, gpu_ctx, synth_pocket, table):
    """A degenerate axis stops the chain at fragment f: found by group 0 (f even) or through the
    exchanged record of the chosen hypothesis (f odd)."""
    batch = io.generate_dataset_batch(20, 6, 8, seed=21)
    xyz = batch.atom_xyz.copy()
    for i in range(8):
        if i % 4 == 3:
            continue
        a0, f0 = int(batch.atom_off[i]), int(batch.frag_off[i])
        b, e = batch.frag_axis[f0 + i % 6]
        xyz[a0 + e] = xyz[a0 + b]
    bad = native.LigandBatch(batch.atom_off, xyz, batch.atom_type, batch.bond_off, batch.bonds, batch.frag_off,
                             batch.frag_axis, batch.frag_mask, list(batch.ids))
    cfg = model.DockConfig()
    dp = gpu_ctx.pocket(synth_pocket, table)
    s, q = _both(monkeypatch, gpu_ctx, dp, bad, cfg, 1)
    o = oracle.dock_batch(bad, synth_pocket, table, cfg, 1)
    assert (o.results["status"][[0, 1, 2, 4, 5, 6]] == native.STATUS_DEGENERATE_AXIS).all()
    _same(s, q, bad)
    compare(bad, s, o, cfg)


def test_auto_mode_spreads_single_ligands(gpu_ctx, synth_pocket, table):
    """Unforced, a one-ligand call with the default 8 restarts runs spread over 8 clusters of 10
    CTAs (80 SMs); a 64-ligand call keeps the one-CTA chain (its clusters would not be resident)."""
    cfg = model.DockConfig()
    dp = gpu_ctx.pocket(synth_pocket, table)
    batch = io.generate_dataset_batch(36, 20, 64, seed=2)
    one = _dock(gpu_ctx, dp, batch.subset([0]), cfg, 0)
    assert one.stats.lat_spread == 10
    many = _dock(gpu_ctx, dp, batch, cfg, 0)
    assert many.stats.lat_spread == 1
    for f in one.results.dtype.names:
        assert one.results[f][0] == many.results[f][0], f
