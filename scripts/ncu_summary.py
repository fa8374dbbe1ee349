"""Key metrics of an `ncu --set full` report as a small text summary (for profiles/).

    python scripts/ncu_summary.py gpurun_out/prof_gemm.ncu-rep > profiles/r01_ncu_gemm.txt
"""
import csv
import io
import subprocess
import sys

KEYS = [
    "Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum.per_second", "dram__bytes_write.sum.per_second",
    "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__m_xbar2l1tex_read_bytes.sum.per_second",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "smsp__inst_executed.sum",
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    for row in rows[2:]:
        print("-" * 80)
        for k in KEYS:
            if k in head:
                i = head.index(k)
                print(f"{k:90s} {row[i]:>20s} {units[i]}")
        stalls = []
        for i, n in enumerate(head):
            if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued"):
                try:
                    stalls.append((float(row[i].replace(",", "")), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        if stalls:
            tot = sum(s for s, _ in stalls) or 1.0
            print("top stall reasons (pc sampling):",
                  ", ".join(f"{n} {100 * s / tot:.0f}%" for s, n in sorted(stalls, reverse=True)[:6]))


if __name__ == "__main__":
    main(sys.argv[1])
