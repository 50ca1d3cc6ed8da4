"""Parity helpers: compare the device outputs with the CPU oracle field by field."""
import numpy as np


def compare(batch, gpu, orc, cfg):
    """Bit-exact comparison of every selected index and score."""
    n, N = batch.n, cfg.restarts_n
    g, o = gpu.results, orc.results
    assert np.array_equal(g["status"], o["status"]), _first(g["status"], o["status"], "status")
    ok = o["status"] == 0
    for f in ("geom_score", "chem_fx", "best_restart", "best_ax", "best_ay", "n_kept"):
        assert np.array_equal(g[f][ok].astype(np.int64), o[f][ok].astype(np.int64)), _first(g[f][ok], o[f][ok], f)
    assert np.array_equal(g["poses_scored"].astype(np.int64), o["poses_scored"]), "poses_scored"
    assert np.array_equal(g["bump_early_exits"].astype(np.int64), o["bump_early_exits"]), "bump_early_exits"
    # pair evaluations of the early-exit scan at moving-row granularity (P14): exact and
    # deterministic in both families
    assert np.array_equal(g["bump_checks"].astype(np.int64), o["bump_checks_rows"]), \
        _first(g["bump_checks"], o["bump_checks_rows"], "bump_checks")
    if gpu.restarts is not None:
        for f in ("align_score", "final_geom", "ax", "ay", "valid", "kept"):
            assert np.array_equal(gpu.restarts[f].astype(np.int64), orc.restarts[f].astype(np.int64)), \
                _first(gpu.restarts[f], orc.restarts[f], "restart." + f)
        assert np.array_equal(gpu.restart_torsion, orc.restart_torsion), "restart torsion indices"
    if gpu.best_coords is not None:
        for i in np.nonzero(ok)[0]:
            a0, a1 = batch.atom_off[i], batch.atom_off[i + 1]
            assert np.array_equal(gpu.best_coords[a0:a1], orc.best_coords[a0:a1]), f"best coords ligand {i}"


def _first(a, b, name):
    a, b = np.asarray(a), np.asarray(b)
    idx = np.nonzero(a.reshape(-1) != b.reshape(-1))[0]
    if len(idx) == 0:
        return name
    i = idx[0]
    return f"{name}: {len(idx)} mismatches, first at {i}: gpu={a.reshape(-1)[i]} oracle={b.reshape(-1)[i]}"
