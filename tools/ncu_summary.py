"""Summarise an ncu --set full report (one or more kernels) as JSON lines of
the metrics DESIGN.md cites.  Usage: python tools/ncu_summary.py rep.ncu-rep"""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "lts__t_bytes.sum": "l2_bytes",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum": "ld_sectors",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum": "ld_requests",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "threads_per_inst",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "smsp__inst_executed.sum": "warp_insts",
    "launch__registers_per_thread": "registers",
    "sm__cycles_active.avg": "sm_active_cycles",
    "sm__cycles_elapsed.avg": "sm_elapsed_cycles",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "lts__t_sectors.sum": "l2_sectors",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed": "l1_throughput_pct",
}
UNIT = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1, "usecond": 1e-6, "msecond": 1e-3,
        "nsecond": 1e-9, "second": 1, "us": 1e-6, "ms": 1e-3, "ns": 1e-9, "s": 1}


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        rec = {"kernel": vals[hdr.index("Kernel Name")][:120]}
        for i, h in enumerate(hdr):
            if h in WANT:
                v = vals[i].replace(",", "")
                try:
                    x = float(v) * UNIT.get(units[i], 1.0)
                except ValueError:
                    x = v
                rec[WANT[h]] = x
        if "dram_read" in rec and "dram_write" in rec:
            rec["dram_traffic_bytes"] = rec["dram_read"] + rec["dram_write"]
        if "ld_sectors" in rec and rec.get("ld_requests"):
            rec["sectors_per_request"] = rec["ld_sectors"] / rec["ld_requests"]
        if rec.get("sm_elapsed_cycles"):
            rec["sm_active_frac"] = rec["sm_active_cycles"] / rec["sm_elapsed_cycles"]
        # duration is in seconds (ncu mixes ms / us units per kernel)
        if isinstance(rec.get("duration"), float) and rec["duration"] > 0:
            rec["duration_ms"] = rec["duration"] * 1e3
            if "dram_traffic_bytes" in rec:
                rec["dram_gbs"] = rec["dram_traffic_bytes"] / rec["duration"] / 1e9
            if isinstance(rec.get("l2_sectors"), float):
                rec["l2_bytes"] = rec["l2_sectors"] * 32
                rec["l2_gbs"] = rec["l2_bytes"] / rec["duration"] / 1e9
        print(json.dumps(rec))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
