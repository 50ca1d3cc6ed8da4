"""Staged device probe: dock growing batches through each entry point, printing (flushed) after
every step so a stall is localised even when the process is killed. Diagnostics only."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_05069_b200 import io, model, native  # noqa: E402


def say(*a):
    print(*a, flush=True)


pocket = io.synthetic_pocket()
table = native.InteractionTable.default()
ctx = native.Context(0)
dp = ctx.pocket(pocket, table)
say("ctx ok")
for L in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "8,200,2000,20000,30000").split(",")]:
    batch = io.generate_mixed_batch(L, seed=3)
    for fam in (native.FAMILY_BATCHED, native.FAMILY_LATENCY):
        if fam == native.FAMILY_LATENCY and L > 2000:
            continue
        t = time.time()
        rb = native.ResidentBatch(ctx, native.pack(batch))
        st = rb.dock(dp, model.DockConfig(), family=fam)
        say(f"resident L={L} fam={fam} align {st.align_ms:.3f} opt {st.optimize_ms:.3f} wall {time.time() - t:.2f}s")
        t = time.time()
        out = ctx.dock(dp, native.pack(batch), model.DockConfig(), family=fam)
        say(f"dock     L={L} fam={fam} wall {time.time() - t:.2f}s")
