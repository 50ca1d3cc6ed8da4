"""Device-side ingest (ds_generate_resident): the GPU generator + packer
must produce exactly the arrays of the host generator + packer (io.generate_batch + pack), and
docking the resident result must give the host path's results."""
import numpy as np
import pytest

from paper_2209_05069_b200 import io, model, native

pytestmark = pytest.mark.gpu


def _host_packed(seed, first, shapes):
    return native.pack(io.generate_batch(shapes, seed, first))


@pytest.mark.parametrize("seed,first", [(5, 0), (11, 123456789), (-3, 7)])
def test_generated_inputs_bit_identical(gpu_ctx, seed, first):
    shapes = io.mixed_shapes(3000, seed, first)
    shapes = np.concatenate([shapes, [[70, 60], [54, 0], [8, 0], [3, 0], [1, 0], [40, 20]]]).astype(np.int32)
    rb = native.ResidentBatch.generated(gpu_ctx, seed, first, shapes)
    xyzt, fd, idh = rb.read_inputs()
    ref = _host_packed(seed, first, shapes)
    assert np.array_equal(rb.atom_off, ref.atom_off) and np.array_equal(rb.frag_off, ref.frag_off)
    assert np.array_equal(xyzt.view(np.uint32), ref.atom_xyzt[:len(xyzt)].view(np.uint32))
    assert np.array_equal(fd, ref.frag_desc[:len(fd)])
    assert np.array_equal(idh, ref.id_hash)
    rb.close()


def test_generated_batch_docks_like_host(gpu_ctx, synth_pocket, table):
    shapes = io.mixed_shapes(2000, 4, 1000)
    dp = gpu_ctx.pocket(synth_pocket, table)
    cfg = model.DockConfig()
    rb = native.ResidentBatch.generated(gpu_ctx, 4, 1000, shapes)
    rb.dock(dp, cfg)
    got = rb.download()
    rb.close()
    host = native.ResidentBatch(gpu_ctx, _host_packed(4, 1000, shapes))
    host.dock(dp, cfg)
    want = host.download()
    host.close()
    assert np.array_equal(got, want)


def test_generator_rejects_infeasible_shape(gpu_ctx):
    with pytest.raises(model.InfeasibleShape):
        native.ResidentBatch.generated(gpu_ctx, 1, 0, np.array([[10, 9]], np.int32))


def test_generate_empty_and_reuse(gpu_ctx, synth_pocket, table):
    """An empty generated batch docks to nothing; a generated batch followed by a host-packed one on
    the same context (shared device buffers) still matches the host path."""
    dp = gpu_ctx.pocket(synth_pocket, table)
    cfg = model.DockConfig()
    rb = native.ResidentBatch.generated(gpu_ctx, 2, 0, np.zeros((0, 2), np.int32))
    assert rb.n == 0
    rb.dock(dp, cfg)
    assert len(rb.download()) == 0
    rb.close()
    shapes = io.mixed_shapes(300, 8, 0)
    g = native.ResidentBatch.generated(gpu_ctx, 8, 0, shapes)
    g.dock(dp, cfg, family=native.FAMILY_LATENCY)
    got = g.download()
    g.close()
    out = gpu_ctx.dock(dp, _host_packed(8, 0, shapes), cfg, 0, native.FAMILY_LATENCY)
    for f in ("status", "geom_score", "chem_fx", "best_restart", "best_ax", "best_ay", "n_kept"):
        assert np.array_equal(got[f], out.results[f]), f
