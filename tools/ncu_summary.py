import csv, sys
rows=list(csv.reader(open(sys.argv[1])))
h=rows[0]; units=rows[1]
for v in rows[2:]:
    name = v[h.index('Kernel Name')] if 'Kernel Name' in h else ''
    print('==', name[:100])
    want=['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','lts__t_bytes.sum','sm__throughput.avg.pct_of_peak_sustained_elapsed',
    'smsp__thread_inst_executed_per_inst_executed.ratio','sm__warps_active.avg.pct_of_peak_sustained_active','smsp__issue_active.avg.pct_of_peak_sustained_active',
    'lts__t_sector_hit_rate.pct','l1tex__t_sector_hit_rate.pct','launch__registers_per_thread','sm__maximum_warps_per_active_cycle_pct',
    'dram__throughput.avg.pct_of_peak_sustained_elapsed','lts__throughput.avg.pct_of_peak_sustained_elapsed','l1tex__throughput.avg.pct_of_peak_sustained_active','launch__grid_size','launch__block_size','smsp__inst_executed.sum',
    'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active','smsp__sass_thread_inst_executed_op_ffma_pred_on.sum','smsp__sass_thread_inst_executed_op_fadd_pred_on.sum','smsp__sass_thread_inst_executed_op_fmul_pred_on.sum','smsp__sass_inst_executed_op_local_ld.sum','smsp__sass_inst_executed_op_local_st.sum']
    for w in want:
        if w in h: i=h.index(w); print(f"  {w:70s} {v[i]} {units[i]}")
    st=[]
    for i,n in enumerate(h):
        if n.startswith('smsp__average_warps_issue_stalled') and n.endswith('per_issue_active.ratio'):
            try: st.append((float(v[i].replace(',','')),n.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio','')))
            except: pass
    print('  stalls/issue:', ', '.join(f"{n} {x:.2f}" for x,n in sorted(st,reverse=True)[:8]))
