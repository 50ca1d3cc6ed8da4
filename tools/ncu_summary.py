"""Summarise an ncu report (read here, on the CPU box) into profiles/: key per-kernel metrics as
JSON + a markdown table, and the per-launch share list from a `--metrics gpu__time_duration.sum`
CSV.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01/ncu_kernels [launches.csv]
"""
import csv
import os
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "smsp__inst_executed.sum": "warp_inst_executed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "pipe_fma_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "pipe_alu_pct",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed": "pipe_fmaheavy_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_wavefront_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "pipe_lsu_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "launch__registers_per_thread": "regs",
    "launch__occupancy_limit_registers": "occ_limit_regs",
    "launch__occupancy_limit_shared_mem": "occ_limit_smem",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "active_threads_per_inst",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio": "stall_long_sb",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio": "stall_short_sb",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio": "stall_not_selected",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio": "stall_math_throttle",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio": "stall_wait",
}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        k = {"kernel": d.get("Kernel Name", "?")}
        for m, name in KEYS.items():
            if m in d:
                try:
                    v = float(d[m].replace(",", ""))
                except ValueError:
                    continue
                unit = u.get(m, "")
                if unit == "Mbyte":
                    v *= 1e6
                elif unit == "Kbyte":
                    v *= 1e3
                elif unit == "Gbyte":
                    v *= 1e9
                elif unit in ("msecond", "ms"):
                    v *= 1e-3
                elif unit in ("usecond", "us"):
                    v *= 1e-6
                elif unit in ("nsecond", "ns"):
                    v *= 1e-9
                k[name] = v
        res.append(k)
    return res


def launches(path):
    rows = []
    with open(path) as fh:
        text = fh.read()
    start = text.find('"ID"')
    for r in csv.DictReader(io.StringIO(text[start:])):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            v = float(r["Metric Value"].replace(",", ""))
            unit = r.get("Metric Unit", "")
            scale = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}.get(unit, 1e-9)
            rows.append((r["Kernel Name"], v * scale))
    tot = sum(v for _, v in rows)
    agg = {}
    for k, v in rows:
        key = k.split("(")[0]
        agg[key] = agg.get(key, 0.0) + v
    return {"launches": len(rows), "total_s": tot,
            "share": {k: {"seconds": v, "share": v / tot if tot else 0.0} for k, v in sorted(agg.items(), key=lambda x: -x[1])}}


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("out")
    ap.add_argument("launch_csv", nargs="?")
    ap.add_argument("--ligands", type=int, default=0, help="ligands docked per profiled launch (per-ligand calibration)")
    ap.add_argument("--workload", default="")
    ap.add_argument("--lib", default="", help="the profiled libdockscreen.so: its sha256[:16] ties the "
                                               "calibration to this build (bench.py checks it)")
    a = ap.parse_args()
    rep, out = a.report, a.out
    doc = {"report": rep, "kernels": raw(rep), "ligands": a.ligands, "workload": a.workload}
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2209_05069_b200.native import source_sha16
    doc["src_sha16"] = source_sha16()   # the tree this summary is made from = the profiled build's
    if a.lib:
        import hashlib
        with open(a.lib, "rb") as fh:
            doc["lib_sha16"] = hashlib.sha256(fh.read()).hexdigest()[:16]
    if a.launch_csv:
        doc["launch_list"] = launches(a.launch_csv)
    with open(out + ".json", "w") as fh:
        json.dump(doc, fh, indent=1)
    lines = ["| kernel | ms | warp-inst | issue % | warps % | fma pipe % | alu pipe % | smem wavefronts | bank conflicts | DRAM B | L2 hit % | regs |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for k in doc["kernels"]:
        lines.append("| %s | %.3f | %.3e | %.1f | %.1f | %.1f | %.1f | %.3e | %.3e | %.3e | %.1f | %d |" % (
            k["kernel"].split("(")[0][:40], 1e3 * k.get("duration", 0), k.get("warp_inst_executed", 0),
            k.get("issue_active_pct", 0), k.get("warps_active_pct", 0), k.get("pipe_fma_pct", 0),
            k.get("pipe_alu_pct", 0), k.get("smem_wavefronts", 0), k.get("smem_bank_conflicts", 0),
            k.get("dram_read", 0) + k.get("dram_write", 0),
            k.get("l2_hit_pct", 0), int(k.get("regs", 0))))
    if "launch_list" in doc:
        lines += ["", "launch list (ncu gpu__time_duration.sum, cold-cache, serialised):", ""]
        for name, v in doc["launch_list"]["share"].items():
            lines.append("- %s: %.3f s total, %.1f %% of device time" % (name[:60], v["seconds"], 100 * v["share"]))
    with open(out + ".md", "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
