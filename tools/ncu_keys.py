"""Print the key counters of an `ncu --page raw --csv` dump, one column per launch."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0]
keys = ['Kernel Name', 'gpu__time_duration.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct',
        'sm__inst_executed_pipe_fp64.avg.pct', 'smsp__inst_executed.sum', 'launch__registers_per_thread', 'launch__occupancy_limit',
        'l1tex__throughput.avg.pct_of_peak_sustained_elapsed', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'dram__throughput.avg.pct', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'l1tex__t_sector_hit_rate', 'lts__t_sector_hit_rate.pct',
        'smsp__average_warps_issue_stalled', 'smsp__average_warp_latency_per_inst_issued', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'local', 'lts__t_sectors_op_read.sum', 'lts__t_sectors_op_write.sum', 'sm__cycles_elapsed.avg ', 'achieved_occupancy', 'sm__maximum_warps']
extra = sys.argv[2:]
for i, h in enumerate(hdr):
    if any(k in h for k in keys + extra):
        vals = [r[i][:42] for r in rows[2:]]
        if all(v in ('0', '', '0.000000') for v in vals) and 'Kernel' not in h:
            continue
        print(f"{h[:95]:95s} {rows[1][i][:10]:10s}", vals)
