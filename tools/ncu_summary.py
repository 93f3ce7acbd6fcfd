"""Summarise an ncu --set full report into a small JSON for profiles/.
    python tools/ncu_summary.py gpurun_out/prof_k_data_r1c.ncu-rep profiles/ncu_C2_data.json [algo_bytes]
"""
import csv, io, json, subprocess, sys

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "sm__inst_executed.avg.per_cycle_active": "ipc_active",
    "smsp__inst_executed.sum": "warp_instructions",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "simt_threads_per_inst",
    "smsp__sass_branch_targets_threads_divergent.sum": "divergent_branch_targets",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__shared_mem_per_block_dynamic": "smem_dynamic_per_block",
    "launch__occupancy_limit_shared_mem": "occupancy_limit_smem_blocks",
    "sm__cycles_elapsed.avg.per_second": "sm_clock_hz",
    "lts__t_bytes.sum": "l2_bytes",
    # shared-memory (MIO) pipe: the binding resource of the tree walks
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed": "l1tex_lsu_wavefronts_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_wavefronts_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum": "smem_ld_wavefronts",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum": "smem_ld_bank_conflicts",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio": "stall_short_scoreboard",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio": "stall_long_scoreboard",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio": "stall_wait",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio": "stall_mio_throttle",
    "sm__cycles_elapsed.avg": "sm_cycles",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9,
        "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1, "second": 1,
        "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "Kbyte/block": 1e3, "byte/block": 1}

def main():
    rep, out = sys.argv[1], sys.argv[2]
    algo_bytes = float(sys.argv[3]) if len(sys.argv) > 3 else None
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    res = {"report": rep.split("/")[-1], "kernels": []}
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:120]}
        for k, name in METRICS.items():
            if k in hdr:
                v = r[hdr.index(k)].replace(",", "")
                u = units[hdr.index(k)]
                try:
                    f = float(v) * UNIT.get(u, 1)
                except ValueError:
                    continue
                d[name] = f
        if "dram_read" in d:
            d["dram_bytes_per_launch"] = d["dram_read"] + d.get("dram_write", 0)
            if algo_bytes:
                d["algorithmic_bytes"] = algo_bytes
                d["traffic_over_algorithmic"] = d["dram_bytes_per_launch"] / algo_bytes
                d["achieved_GBs_under_ncu"] = algo_bytes / d["duration"] / 1e9
        if "smem_wavefronts" in d and d.get("sm_cycles"):
            # shared-memory wavefronts per SM-cycle (the pipe retires <= 1 per cycle)
            sms = 148.0
            d["shared_wavefronts_per_clk_per_sm"] = d["smem_wavefronts"] / (d["sm_cycles"] * sms)
            if "smem_ld_bank_conflicts" in d and d.get("smem_ld_wavefronts"):
                d["shared_conflict_fraction"] = d["smem_ld_bank_conflicts"] / d["smem_ld_wavefronts"]
        res["kernels"].append(d)
    k0 = res["kernels"][0]
    res.update({k: k0[k] for k in ("dram_bytes_per_launch", "duration") if k in k0})
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))

main()
