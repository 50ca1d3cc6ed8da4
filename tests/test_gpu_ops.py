"""The L2 ops of the native slot on the device (ds_op_*, the `kernels` module) against the CPU
oracle, bit for bit, at SPEC acceptance scale (10^4 transforms)."""
import numpy as np
import pytest

import oracle
from paper_2209_05069_b200 import io, kernels, model, native

pytestmark = pytest.mark.gpu


def _poses(rng, P, n, scale=6.0):
    return rng.uniform(-scale, scale, size=(P, n, 3)).astype(np.float32)


def test_apply_rigid_bit_exact_1e4():
    rng = np.random.default_rng(40)
    x = _poses(rng, 10_000, 24)
    m = np.stack([kernels.rot_y(int(a)) @ kernels.rot_x(int(b)) for a, b in rng.integers(0, 360, size=(10_000, 2))])
    c = rng.uniform(-3, 3, size=(10_000, 3)).astype(np.float32)
    g = kernels.apply_rigid(x, m, c)
    o = oracle.apply_rigid(x, m, c)
    assert np.array_equal(g.view(np.uint32), o.view(np.uint32))
    # SPEC.md:141 identity -> unchanged, up to the rounding of (p - c) + c (<= 1 ulp)
    ident = kernels.apply_rigid(x[0], np.eye(3), c[0])
    assert (np.abs(ident - x[0]) <= np.spacing(np.abs(x[0]) + np.abs(c[0]))).all()


@pytest.mark.parametrize("deg", [0, 36, 144, 300, 17])
def test_apply_torsion_bit_exact_1e4(deg):
    rng = np.random.default_rng(41 + deg)
    n = 40
    x = _poses(rng, 2000, n)
    mask = frozenset(rng.choice(np.arange(2, n), size=17, replace=False).tolist())
    frag = model.Fragment(0, 1, mask)
    g = kernels.apply_torsion(x, frag, deg)
    o, st = oracle.apply_torsion(x, 0, 1, mask, deg)
    assert (st == 0).all()
    assert np.array_equal(g.view(np.uint32), o.view(np.uint32))
    fixed = [i for i in range(n) if i not in mask]
    assert np.array_equal(g[:, fixed].view(np.uint32), x[:, fixed].view(np.uint32))
    if deg == 0:
        assert np.array_equal(g.view(np.uint32), x.view(np.uint32))


def test_apply_torsion_degenerate_axis():
    x = _poses(np.random.default_rng(3), 4, 10)
    x[2, 1] = x[2, 0]
    with pytest.raises(model.DegenerateAxis):
        kernels.apply_torsion(x, model.Fragment(0, 1, frozenset({4, 5})), 36)
    with pytest.raises(model.MalformedFragment):
        kernels.apply_torsion(x, model.Fragment(0, 1, frozenset({1, 5})), 36)


@pytest.mark.parametrize("early_exit", [True, False])
def test_bump_check_matches_oracle_and_counts(early_exit):
    rng = np.random.default_rng(42)
    x = rng.uniform(-4, 4, size=(3000, 40, 3)).astype(np.float32)
    mask = frozenset(range(10, 40))
    frag = model.Fragment(5, 9, mask)
    c = model.Counters()
    g = kernels.bump_check(x, frag, 0.8, early_exit, c)
    ob, op = oracle.bump_check(x, 5, 9, mask, 0.8, early_exit)
    assert np.array_equal(g, ob)
    assert c.bump_checks == int(op.sum())
    assert c.bump_early_exits == (int(ob.sum()) if early_exit else 0)
    assert kernels.bump_check(np.zeros((12, 3), np.float32), model.Fragment(0, 1, frozenset({2})), 0.8)


def test_grid_score_and_rescore_ops_match_oracle(synth_pocket, table):
    rng = np.random.default_rng(43)
    lo = np.array(synth_pocket.grid_origin, np.float32)
    hi = lo + np.float32(synth_pocket.grid_spacing) * (np.array(synth_pocket.grid_dims, np.float32) - 1)
    x = rng.uniform(lo - 2, hi + 2, size=(500, 30, 3)).astype(np.float32)   # some atoms outside: -100
    types = rng.integers(0, 16, size=30).astype(np.uint8)
    g = kernels.grid_score(x, synth_pocket)
    assert [int(v) for v in g] == [oracle.grid_score(synth_pocket, table, p) for p in x]
    fx = kernels.rescore_fx(x[:60], types, synth_pocket, table)
    assert [int(v) for v in fx] == [oracle.rescore_fx(synth_pocket, table, p, types) for p in x[:60]]
    assert kernels.rescore(x[0], types, synth_pocket, table) == float(fx[0]) / 2 ** 24


def test_rot_matches_oracle():
    for d in (0, 12, 90, 180, 270, 359):
        assert np.array_equal(kernels.rot_x(d), oracle.rot(0, d))
        assert np.array_equal(kernels.rot_y(d), oracle.rot(1, d))


def test_stale_resident_batch_fails_loudly(gpu_ctx, synth_pocket, table):
    """A resident batch handle whose context buffers were reused by a later upload / ds_dock call
    is rejected (DS_ERR_INVALID_ARG) instead of silently docking or downloading another batch's
    data; op calls do not invalidate it."""
    from paper_2209_05069_b200.native import ResidentBatch, pack
    cfg = model.DockConfig()
    dp = gpu_ctx.pocket(synth_pocket, table)
    a = ResidentBatch(gpu_ctx, pack(io.generate_mixed_batch(50, seed=1)))
    a.dock(dp, cfg)
    kernels.grid_score(np.zeros((5, 3), np.float32), synth_pocket)   # other ctx (thread context): no effect
    a.download()
    b = ResidentBatch(gpu_ctx, pack(io.generate_mixed_batch(40, seed=2)))
    with pytest.raises(ValueError, match="stale"):
        a.dock(dp, cfg)
    with pytest.raises(ValueError, match="stale"):
        a.download()
    b.dock(dp, cfg)
    gpu_ctx.dock(dp, pack(io.generate_mixed_batch(10, seed=3)), cfg)
    with pytest.raises(ValueError, match="stale"):
        b.download()
    a.close()
    b.close()
    dp.close()
