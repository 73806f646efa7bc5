"""Summarise an ncu report (--set full) into the metrics DESIGN.md/bench use.
python tools/ncu_summary.py report.ncu-rep [label] > profiles/<name>.txt"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__thread_inst_executed_per_inst_executed.ratio",
    "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "launch__shared_mem_per_block_static", "launch__occupancy_limit_shared_mem",
    "lts__t_requests_op_red.sum", "lts__t_requests_op_atom.sum", "lts__t_sectors_op_red.sum",
    "lts__t_sectors_op_atom.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__sass_inst_executed_op_shared_atom.sum", "smsp__sass_inst_executed_op_global_red.sum",
    "smsp__sass_inst_executed_op_global_atom.sum",
]


def main():
    rep = sys.argv[1]
    label = sys.argv[2] if len(sys.argv) > 2 else rep
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full summary: {label}")
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"\n## kernel: {name[:160]}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"{k:60s} {r[i]:>22s} {units[i]}")
        st = []
        for i, h in enumerate(hdr):
            if "average_warps_issue_stalled" in h and h.endswith("per_issue_active.ratio"):
                try:
                    st.append((float(r[i].replace(",", "")), h))
                except ValueError:
                    pass
        print("top stall reasons (warps stalled per issue):")
        for v, h in sorted(st, reverse=True)[:6]:
            print(f"  {v:8.2f}  {h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}")


if __name__ == "__main__":
    main()
