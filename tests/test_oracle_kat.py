"""The CPU oracle against every known-answer example SPEC.md states for the hot path.

The reference ships no tests or golden vectors; these SPEC examples are the
only reference-side answers that exist, so they pin the oracle (together with the
pure-Python cross-check in test_oracle_crosscheck.py).
"""
import numpy as np
import pytest

import oracle
import pyoracle as py
from paper_2209_05069_b200 import io, model
from paper_2209_05069_b200.native import InteractionTable, LigandBatch

f32 = np.float32


def unit_pocket(values, dims, atoms=(), bins=None, table=None):
    """Grid with origin 0 and spacing 1: the grid frame equals the Å frame."""
    p = model.Pocket((0.0, 0.0, 0.0), 1.0, dims, np.asarray(values, np.int32).reshape(-1), tuple(atoms))
    t = table if table is not None else InteractionTable(np.ones((16, 16), np.float32), bins or ((2.0, 1.0), (8.0, 1.0)))
    return p, t


# ---- transform -------------------------------------------------------
def test_rot_x_known_answers():
    assert np.array_equal(oracle.rot(0, 0), np.eye(3, dtype=np.float32))
    assert np.allclose(oracle.rot(0, 360), np.eye(3), atol=1e-9)
    assert np.allclose(oracle.rot(0, 90) @ np.array([0, 1, 0], np.float32), [0, 0, 1], atol=1e-9)


def test_rot_y_known_answers():
    assert np.array_equal(oracle.rot(1, 0), np.eye(3, dtype=np.float32))
    assert np.allclose(oracle.rot(1, 180) @ np.array([1, 0, 0], np.float32), [-1, 0, 0], atol=1e-9)  # :132
    assert np.allclose(oracle.rot(1, 90) @ np.array([0, 0, 1], np.float32), [1, 0, 0], atol=1e-9)    # :133


@pytest.mark.parametrize("axis", [0, 1, 2])
def test_rotations_orthonormal(axis):
    for d in range(0, 360, 7):
        R = oracle.rot(axis, d).astype(np.float64)
        assert np.allclose(R.T @ R, np.eye(3), atol=1e-6) and abs(np.linalg.det(R) - 1) < 1e-6


def test_rotation_composition():
    """apply_rigid with rot_x(a)·rot_x(b) equals sequential application within 1e-6."""
    rng = np.random.default_rng(0)
    p = rng.normal(size=(20, 3)).astype(np.float32)
    for a, b in [(12, 24), (90, 180), (36, 348)]:
        Rab = np.array(py.mat3_mul(py.rot_x(a), py.rot_x(b)), np.float64).reshape(3, 3)
        seq = (oracle.rot(0, a).astype(np.float64) @ (oracle.rot(0, b).astype(np.float64) @ p.T)).T
        assert np.allclose((Rab @ p.T).T, seq, atol=1e-6)


def test_torsion_angle_zero_and_rigidity():
    rng = np.random.default_rng(1)
    L = py.Ligand("t", rng.normal(scale=2.0, size=(12, 3)).astype(np.float32), [1] * 12, [(0, 1)], [set(range(2, 7))])
    U = [list(d) for d in L.d]
    same = py.torsion(L, 0, U, 0, f32(1e-9))
    assert all(np.array_equal(np.array(a, np.float32), np.array(b, np.float32)) for a, b in zip(same, U))  # :151
    for deg in (36, 144, 252):
        out = py.torsion(L, 0, U, deg, f32(1e-9))
        X, Y = np.array(U, np.float64), np.array(out, np.float64)
        fixed = [i for i in range(12) if i not in L.masks[0]]
        assert np.array_equal(X[fixed], Y[fixed])                                                        # :152
        M = sorted(L.masks[0])
        for part in (M, fixed):
            dx = np.linalg.norm(X[part][:, None] - X[part][None], axis=-1)
            dy = np.linalg.norm(Y[part][:, None] - Y[part][None], axis=-1)
            assert np.allclose(dx, dy, rtol=1e-6, atol=1e-6)                                             # :153
        back = py.torsion(L, 0, out, (360 - deg) % 360, f32(1e-9))
        assert np.allclose(np.array(back, np.float64), X, atol=1e-5)                                     # :156


def test_torsion_degenerate_axis():
    L = py.Ligand("t", np.zeros((4, 3), np.float32), [1] * 4, [(0, 1)], [{2, 3}])
    assert py.torsion(L, 0, [list(d) for d in L.d], 36, f32(1e-9)) is None                               # :149


# ---- scoring ---------------------------------------------------------
def test_grid_score_known_answers():
    p, t = unit_pocket(np.zeros(27), (3, 3, 3))
    assert oracle.grid_score(p, t, np.array([[1.2, 0.4, 1.9]], np.float32)) == 0                        # :189
    vals = np.zeros(27, np.int32)
    vals[1 + 3 * (2 + 3 * 1)] = 7
    p, t = unit_pocket(vals, (3, 3, 3))
    assert oracle.grid_score(p, t, np.array([[1.0, 2.0, 1.0]], np.float32)) == 7                         # :190
    assert oracle.grid_score(p, t, np.array([[9.0, 2.0, 1.0]], np.float32)) == -100                      # :186


def test_grid_score_brute_force():
    """random 4x4x4 grid, 5 atoms == brute-force nearest-node summation."""
    rng = np.random.default_rng(2)
    for _ in range(20):
        vals = rng.integers(-10, 11, size=64).astype(np.int32)
        p, t = unit_pocket(vals, (4, 4, 4))
        x = rng.uniform(-0.49, 3.49, size=(5, 3)).astype(np.float32)
        nodes = np.stack(np.meshgrid(np.arange(4), np.arange(4), np.arange(4), indexing="ij"), -1).reshape(-1, 3)
        want = 0
        for a in x:
            n = nodes[np.argmin(((nodes - a.astype(np.float64)) ** 2).sum(1))]
            want += int(vals[n[0] + 4 * (n[1] + 4 * n[2])])
        assert oracle.grid_score(p, t, x) == want


def test_grid_score_translation_covariant():
    """Shifting pose and grid origin by the same vector leaves the score unchanged."""
    rng = np.random.default_rng(3)
    vals = rng.integers(-10, 11, size=125).astype(np.int32)
    x = rng.uniform(0.1, 3.9, size=(8, 3)).astype(np.float32)
    p0 = model.Pocket((0.0, 0.0, 0.0), 1.0, (5, 5, 5), vals)
    p1 = model.Pocket((2.0, -3.0, 4.0), 1.0, (5, 5, 5), vals)
    t = InteractionTable.default()
    assert oracle.grid_score(p0, t, x) == oracle.grid_score(p1, t, x + np.array([2, -3, 4], np.float32))


def test_bump_known_answers_and_early_exit_equivalence():
    L = py.Ligand("b", np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0], [2, 0, 0]], np.float32), [1] * 4, [(0, 1)], [{2}])
    U = [list(d) for d in L.d]
    assert py.bump(L, 0, U, f32(0.64))                                                              # :199
    L2 = py.Ligand("b", np.array([[0, 0, 0], [1, 0, 0], [5, 0, 0], [9, 0, 0]], np.float32), [1] * 4, [(0, 1)], [{2}])
    assert not py.bump(L2, 0, [list(d) for d in L2.d], f32(0.64))                                   # :200
    # random 40-atom ligands: result equals an all-pairs numpy scan
    rng = np.random.default_rng(4)
    for _ in range(10):
        x = rng.uniform(0, 6, size=(40, 3)).astype(np.float32)
        mask = set(rng.choice(np.arange(2, 40), size=12, replace=False).tolist())
        L3 = py.Ligand("r", x, [1] * 40, [(0, 1)], [mask])
        U3 = np.array([list(d) for d in L3.d], np.float64)
        comp = [j for j in range(40) if j not in mask and j not in (0, 1)]
        d2 = ((U3[sorted(mask)][:, None] - U3[comp][None]) ** 2).sum(-1)
        if np.any(np.abs(d2 - 0.64) < 1e-4):
            continue  # too close to the threshold for an f64 reference
        assert py.bump(L3, 0, [list(d) for d in L3.d], f32(0.64)) == bool((d2 < 0.64).any())


def test_rescore_known_answers():
    p, t = unit_pocket(np.zeros(8), (2, 2, 2))
    assert oracle.rescore_fx(p, t, np.zeros((3, 3), np.float32), np.ones(3, np.uint8)) == 0         # :209 empty pocket
    p, t = unit_pocket(np.zeros(8), (2, 2, 2), atoms=[model.Atom.of(100.0, 0.0, 0.0, 1)])
    assert oracle.rescore_fx(p, t, np.zeros((1, 3), np.float32), np.ones(1, np.uint8)) == 0         # :210 beyond cutoff
    # 3 ligand atoms x 2 pocket atoms, unit weights, bins (2 Å: x1.0, 8 Å: x1.0): every pair < 8 Å counts 1
    p, t = unit_pocket(np.zeros(8), (2, 2, 2), atoms=[model.Atom.of(0, 0, 0, 1), model.Atom.of(3, 0, 0, 2)])
    lig = np.array([[0, 1, 0], [1, 1, 1], [6, 0, 0]], np.float32)
    want = sum(1 for a in lig for b in ([0, 0, 0], [3, 0, 0]) if np.sum((a - np.array(b)) ** 2) < 64)
    assert oracle.rescore_fx(p, t, lig, np.ones(3, np.uint8)) == want * (1 << 24)                    # :211


def test_rescore_relabel_symmetry():
    """Swapping two identical-type atoms leaves the score unchanged exactly."""
    pocket = io.synthetic_pocket()
    t = InteractionTable.default()
    rng = np.random.default_rng(5)
    x = rng.uniform(-6, 6, size=(10, 3)).astype(np.float32)
    ty = np.full(10, 3, np.uint8)
    a = oracle.rescore_fx(pocket, t, x, ty)
    assert a == oracle.rescore_fx(pocket, t, x[::-1].copy(), ty)


# ---- docking ---------------------------------------------------------
def _one(lig_xyz, types, frags, lid="k"):
    atoms = tuple(model.Atom.of(*p, int(t)) for p, t in zip(lig_xyz, types))
    n = len(atoms)
    bonds = tuple((i, i + 1) for i in range(n - 1))
    fr = tuple(model.Fragment(b, e, frozenset(m)) for b, e, m in frags)
    return model.Ligand(lid, atoms, bonds, fr)


def test_starting_pose_determinism_and_degenerate_grid():
    P = py.Pocket((0, 0, 0), 1.0, (9, 9, 9), np.zeros(729), [], [], np.ones(256), ((8.0, 1.0),))
    L = py.Ligand("lig", np.random.default_rng(6).normal(size=(5, 3)).astype(np.float32), [1] * 5, [], [])
    a = py.starting_pose(L, P, 0, 0)
    assert a == py.starting_pose(L, P, 0, 0)                                                        # :243
    assert a[1] != py.starting_pose(L, P, 1, 0)[1]                                                  # :244
    P1 = py.Pocket((0, 0, 0), 1.0, (1, 1, 1), np.zeros(1), [], [], np.ones(256), ((8.0, 1.0),))
    assert all(float(x) == 0.0 for x in py.starting_pose(L, P1, 3, 0)[1])                           # :245


def test_rigid_ligand_uniform_grid_restart0_at_00():
    """rigid ligand (0 fragments) in a uniform grid: best pose = restart 0 at (0,0);
    align in a uniform grid returns (0,0) and scores 900 poses per restart."""
    pocket = model.Pocket((-20.0, -20.0, -20.0), 1.0, (41, 41, 41), np.full(41 ** 3, 3, np.int32), ())
    t = InteractionTable.default()
    lig = _one(np.array([[0, 0, 0], [1.5, 0, 0], [1.5, 1.5, 0]], np.float32), [1, 2, 3], [])
    b = LigandBatch.from_ligands([lig])
    cfg = model.DockConfig()
    out = oracle.dock_batch(b, pocket, t, cfg)
    r = out.results[0]
    assert r["status"] == 0 and r["best_restart"] == 0 and (r["best_ax"], r["best_ay"]) == (0, 0)
    assert (out.restarts["ax"] == 0).all() and (out.restarts["ay"] == 0).all()
    assert r["poses_scored"] == 8 * 900
    assert r["geom_score"] == 9


def test_counter_law_and_fragment_evaluations():
    """poses_scored = N x 900 + 10 x F per restart."""
    pocket = io.synthetic_pocket()
    t = InteractionTable.default()
    b = io.generate_dataset_batch(16, 12, 4, seed=9)
    out = oracle.dock_batch(b, pocket, t, model.DockConfig())
    assert (out.results["poses_scored"] == 8 * (900 + 10 * 12)).all()
    b0 = io.generate_dataset_batch(10, 0, 4, seed=9)
    out0 = oracle.dock_batch(b0, pocket, t, model.DockConfig())
    assert (out0.restarts["align_score"] == out0.restarts["final_geom"]).all()                      # :263


def test_early_exit_purity():
    """early_exit changes counters only, never scores or poses."""
    pocket = io.synthetic_pocket()
    t = InteractionTable.default()
    b = io.generate_mixed_batch(40, seed=10)
    on = oracle.dock_batch(b, pocket, t, model.DockConfig(early_exit=True))
    off = oracle.dock_batch(b, pocket, t, model.DockConfig(early_exit=False))
    for f in ("status", "geom_score", "chem_fx", "best_restart", "best_ax", "best_ay", "poses_scored"):
        assert np.array_equal(on.results[f], off.results[f])
    assert np.array_equal(on.restart_torsion, off.restart_torsion)
    assert np.array_equal(on.best_coords, off.best_coords)
    assert (on.results["bump_checks"] <= off.results["bump_checks"]).all()
    assert (on.results["bump_checks"] < off.results["bump_checks"]).any()
    assert (on.results["bump_early_exits"] <= on.results["bump_checks"]).all()


def test_restart_order_independence():
    """Permuting restart evaluation order never changes the selection: the
    selection is a function of per-restart records only, so re-selecting from the recorded
    restarts in reversed order reproduces the oracle's choice."""
    pocket = io.synthetic_pocket()
    t = InteractionTable.default()
    b = io.generate_mixed_batch(20, seed=12)
    out = oracle.dock_batch(b, pocket, t, model.DockConfig())
    for i in range(b.n):
        rr = out.restarts[i]
        valid = [r for r in reversed(range(8)) if rr[r]["valid"]]
        order = sorted(valid, key=lambda r: (-rr[r]["final_geom"], r))
        kept = [r for r in order if rr[r]["kept"]]
        assert sorted(kept, key=lambda r: rr[r]["kept"]) == [r for r in order if r in kept]


def test_select_identical_poses_keeps_one():
    """all poses identical -> exactly 1 kept: a single-atom ligand in a uniform grid
    aligns every restart onto its own centre; with one heavy atom all RMSDs between restarts are
    the distances of the centres, so use a 1x1x1 grid where every centre is the origin."""
    pocket = model.Pocket((0.0, 0.0, 0.0), 1.0, (1, 1, 1), np.zeros(1, np.int32), ())
    t = InteractionTable.default()
    lig = _one(np.array([[0, 0, 0]], np.float32), [5], [])
    out = oracle.dock_batch(LigandBatch.from_ligands([lig]), pocket, t, model.DockConfig())
    assert out.results[0]["status"] == 0 and out.results[0]["n_kept"] == 1


def test_select_distant_top4():
    """mutually distant poses, K=4, 8 valid -> the top 4 by score are kept."""
    pocket = io.synthetic_pocket()
    t = InteractionTable.default()
    b = io.generate_dataset_batch(30, 0, 6, seed=13)
    out = oracle.dock_batch(b, pocket, t, model.DockConfig())
    for i in range(b.n):
        rr = out.restarts[i]
        order = sorted(range(8), key=lambda r: (-rr[r]["final_geom"], r))
        kept = sorted([r for r in range(8) if rr[r]["kept"]], key=lambda r: rr[r]["kept"])
        assert kept == order[:4]
