"""Key raw metrics + stall breakdown of every kernel in an ncu report (csv from --page raw --csv)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0]
keys = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'launch__registers_per_thread', 'launch__occupancy_limit_shared_mem', 'launch__occupancy_limit_registers',
        'launch__grid_size', 'smsp__inst_executed.sum', 'lts__t_bytes.sum', 'lts__t_sectors_srcunit_tex_op_write.sum',
        'lts__t_sectors_srcunit_tex_op_read.sum', 'sm__cycles_elapsed.avg', 'lts__throughput.avg.pct_of_peak_sustained_elapsed']
for r in rows[2:]:
    d = dict(zip(hdr, r))
    for k in keys:
        if k in d: print(f"  {k:60s} {d[k]}")
    out = []
    for k in hdr:
        if k.startswith('smsp__average_warps_issue_stalled_') and k.endswith('per_issue_active.ratio'):
            try: out.append((float(d[k]), k))
            except ValueError: pass
    for v, k in sorted(out, reverse=True)[:8]:
        print('   %.3f %s' % (v, k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')))
