"""Print the handful of counters DESIGN.md quotes from an `ncu --page raw --csv`
export.  Usage: python tools/ncu_keys.py raw.csv [row]"""
import csv
import sys

KEYS = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "lts__t_sectors_op_read.sum", "lts__t_sectors_srcunit_tex_op_read.sum", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__warps_eligible.avg.per_cycle_active",
        "l1tex__data_pipe_lsu_wavefronts.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__inst_executed.sum", "l1tex__m_xbar2l1tex_read_sectors.sum")
rows = [r for r in csv.reader(open(sys.argv[1])) if r]
h = next(i for i, r in enumerate(rows) if r[0] == "ID")
names, units = rows[h], rows[h + 1]
for data in rows[h + 2:]:
    print("==", data[names.index("Kernel Name")][:90])
    for n, u, v in zip(names, units, data):
        if n in KEYS:
            print(f"  {n:64s} {v:>18s} {u}")
