"""BASELINE config 5 as a screen: a synthetic ligand database docked across the GPUs of one node,
one process per GPU (torchrun), and the per-ligand best results gathered to rank 0.

    python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port 29531 tools/screen.py --ligands 10000000
    python tools/screen.py --ligands 1000000          # single process, GPU 0

Each rank takes a contiguous slice of the global index space (shard.shard_range), generates it
locally from the global index (so every rank's shard is the same ligands a single-rank run would
dock), docks it through ds_dock (chunked H2D / compute / D2H pipeline) and the fixed-size result
records plus best poses' scores are gathered to rank 0 (shard.gather_records).  Nothing is
exchanged while docking.  Rank 0 prints one JSON line: ligands, wall-clock throughput of the
whole screen (generation excluded), the max per-rank docking time, and the top hits by
chemical score.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--ligands", type=int, default=1_000_000)
ap.add_argument("--seed", type=int, default=5)
ap.add_argument("--top", type=int, default=10)
ap.add_argument("--device-gen", action="store_true",
                help="generate + pack the shard on the GPU (ds_generate_resident) instead of on the host")
a = ap.parse_args()

rank = int(os.environ.get("RANK", "0"))
world = int(os.environ.get("WORLD_SIZE", "1"))
local = int(os.environ.get("LOCAL_RANK", "0"))
local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
if local_world > 1 and "OMP_NUM_THREADS" not in os.environ:
    os.environ["OMP_NUM_THREADS"] = str(max(1, (os.cpu_count() or 1) // local_world))

import torch  # noqa: E402

from paper_2209_05069_b200 import io, model, native, shard  # noqa: E402

dist = None
ndev = torch.cuda.device_count()
device = local % max(ndev, 1)
if world > 1:
    import torch.distributed as dist
    torch.cuda.set_device(device)
    dist.init_process_group("nccl" if ndev >= world else "gloo")

lo, hi = shard.shard_range(a.ligands, world, rank)
ctx = native.Context(device)
dp = ctx.pocket(io.synthetic_pocket(), native.InteractionTable.default())
cfg = model.DockConfig()
t_gen = t_gen_dev = 0.0
if a.device_gen:
    # device-side ingest: only the (heavy, F) shapes are made on the host; the ligands are generated
    # and packed where they are docked, so the timed screen covers generation + docking
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    shapes = io.mixed_shapes(hi - lo, a.seed, lo)
    rb = native.ResidentBatch.generated(ctx, a.seed, lo, shapes)
    st = rb.dock(dp, cfg)
    res = rb.download()
    rb.close()
    t_dock = time.perf_counter() - t0
    device_s = (st.total_ms + rb.generate_ms) / 1e3
    t_gen_dev = rb.generate_ms / 1e3
else:
    t0 = time.perf_counter()
    batch = io.generate_mixed_batch(hi - lo, seed=a.seed, first_index=lo)
    packed = native.pack(batch, pinned=True)
    t_gen = time.perf_counter() - t0
    bufs = native.OutputBuffers(packed, pinned=True)
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    out = ctx.dock(dp, packed, cfg, 0, native.FAMILY_BATCHED, coords=True, buffers=bufs)
    t_dock = time.perf_counter() - t0
    res = out.results
    device_s = out.stats.total_ms / 1e3
if dist is not None:
    dist.barrier()
t_all = time.perf_counter() - t0

recs = shard.gather_records(res, rank, world)
times = shard.gather_records(np.array([t_dock, device_s], np.float64), rank, world)
if rank == 0:
    ok = recs["status"] == 0
    chem = recs["chem_fx"].astype(np.float64) * 2.0 ** -24
    order = np.argsort(-np.where(ok, chem, -np.inf), kind="stable")[:a.top]
    line = {"workload": "config5 screen: mixed config-3 ligands (heavy U{8..40}, F U{0..20}), synthetic pocket"
                        + (", generated + packed on the GPU (timed)" if a.device_gen else ", host-generated (untimed)"),
            "ligands": int(len(recs)), "ranks": world, "ok_frac": float(ok.mean()),
            "screen_s": t_all, "ligands_per_s": len(recs) / t_all,
            "max_rank_dock_s": float(times[0::2].max()), "max_rank_device_s": float(times[1::2].max()),
            "generation_s_rank0": t_gen, "generation_device_s_rank0": t_gen_dev,
            "top_hits": [{"index": int(i), "chem": float(chem[i]), "geom": int(recs["geom_score"][i])} for i in order]}
    print(json.dumps(line), flush=True)
if dist is not None:
    dist.destroy_process_group()
