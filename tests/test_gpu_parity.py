"""GPU parity: the sm_100a kernels against the CPU oracle, bit-exact."""
import numpy as np
import pytest

import oracle
from helpers import compare
from paper_2209_05069_b200 import io, model
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


def test_batched_parity_no_early_exit(gpu_ctx, synth_pocket, table):
    batch = io.generate_mixed_batch(64, seed=4)
    cfg = model.DockConfig(early_exit=False)
    g, o = _run(gpu_ctx, batch, synth_pocket, table, cfg)
    compare(batch, g, o, cfg)
    assert np.array_equal(g.results["bump_checks"].astype(np.int64), o.results["bump_checks"])
