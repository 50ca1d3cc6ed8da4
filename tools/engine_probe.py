import sys, time
sys.path.insert(0, '.')
from paper_2209_05069_b200 import io, model, engines
from paper_2209_05069_b200.native import InteractionTable
pocket = io.synthetic_pocket(); table = InteractionTable.default()
b = io.generate_mixed_batch(20000, seed=3)
t0 = time.perf_counter(); ligs = b.to_ligands(); t1 = time.perf_counter()
print("to_ligands %.2f s" % (t1 - t0))
for w in (1, 8):
    rep = engines.batched_engine.run(ligs, pocket, model.DockConfig(), workers=w, table=table)
    print("batched workers=%d wall %.2f s throughput %.0f/s" % (w, rep.wall_time, rep.throughput))
rep = engines.latency_engine.run(ligs[:2000], pocket, model.DockConfig(), workers=8, table=table)
print("latency 2000 ligands workers=8 wall %.2f s throughput %.0f/s" % (rep.wall_time, rep.throughput))
