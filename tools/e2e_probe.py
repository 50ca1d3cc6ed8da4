"""Where the end-to-end time of a large ds_dock call goes: host wall clock vs the device span
(first H2D .. last D2H, CUDA events) vs the kernels (resident batch)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_05069_b200 import io, model, native  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
batch = io.generate_mixed_batch(n, seed=3)
packed = native.pack(batch, pinned=True)
ctx = native.Context(0)
dp = ctx.pocket(io.synthetic_pocket(), native.InteractionTable.default())
cfg = model.DockConfig()
bufs = native.OutputBuffers(packed, pinned=True)
for _ in range(2):
    ctx.dock(dp, packed, cfg, 0, native.FAMILY_BATCHED, coords=True, buffers=bufs)
for _ in range(3):
    t0 = time.perf_counter()
    o = ctx.dock(dp, packed, cfg, 0, native.FAMILY_BATCHED, coords=True, buffers=bufs)
    wall = 1e3 * (time.perf_counter() - t0)
    print(f"wall {wall:.2f} ms  device span {o.stats.total_ms:.2f} ms  align {o.stats.align_ms:.2f}  "
          f"optimize {o.stats.optimize_ms:.2f}")
rb = native.ResidentBatch(ctx, packed)
st = rb.dock(dp, cfg)
st = rb.dock(dp, cfg)
print(f"resident kernels {st.total_ms:.2f} ms")
