"""Summarise an .ncu-rep (raw page) into the metrics the roofline/DESIGN notes cite.
Usage: python tools/ncu_summary.py <file.ncu-rep> [> profiles/<name>.txt]"""
import csv
import io
import subprocess
import sys

WANT = [
    "Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    tensor_cols = ["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
                   "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
                   "sm__ops_path_tensor_src_tf32_dst_fp32.avg.pct_of_peak_sustained_elapsed",
                   "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active"]
    stall_cols = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_")
                  and h.endswith("per_issue_active.ratio")]
    for r in rows[2:]:
        print("-" * 80)
        for w in WANT + [c for c in tensor_cols if c not in WANT]:
            if w in hdr:
                i = hdr.index(w)
                print(f"{w:70s} {r[i]} {units[i]}")
        st = sorted(((float(r[hdr.index(c)] or 0), c) for c in stall_cols), reverse=True)[:6]
        print("top stall reasons (warps per issue-active cycle):")
        for v, c in st:
            name = c.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")
            print(f"  {name:30s} {v:.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
