"""Compare selected metrics of `ncu --page raw --csv` exports side by side.
Usage: python tools/ncu_cmp.py a.csv b.csv ..."""
import csv
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sectors_srcunit_tex_op_read.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_lg_throttle",
        "smsp__pcsamp_warps_issue_stalled_mio_throttle", "lts__average_gcomp_input_sector_success_rate.pct",
        "lts__t_sectors_srcunit_tex_lookup_miss.sum", "lts__d_sectors_fill_sysmem.sum"]


def load(p):
    rows = list(csv.reader(open(p)))
    h, units, v = rows[0], rows[1], rows[2]
    return {k: (x, u) for k, u, x in zip(h, units, v)}


cols = [load(p) for p in sys.argv[1:]]
print("metric".ljust(58), *[p.split("/")[-1][:18].rjust(18) for p in sys.argv[1:]])
for m in WANT:
    if any(m in c for c in cols):
        print(m[:58].ljust(58), *[(c.get(m, ("-", ""))[0] + " " + c.get(m, ("", ""))[1])[:18].rjust(18) for c in cols])
