import csv, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu","-i",rep,"--page","raw","--csv"],capture_output=True,text=True).stdout
rows=list(csv.reader(raw.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
want=['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed','sm__throughput.avg.pct_of_peak_sustained_elapsed','sm__warps_active.avg.per_cycle_active','launch__registers_per_thread','smsp__inst_executed.sum','sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active','smsp__average_warp_latency_per_inst_issued.ratio','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum','lts__t_bytes.sum','smsp__issue_active.avg.pct_of_peak_sustained_active','launch__grid_size','launch__block_size','launch__shared_mem_per_block_dynamic','sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active','sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed','l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','sm__memory_throughput.avg.pct_of_peak_sustained_elapsed','l1tex__throughput.avg.pct_of_peak_sustained_active']
for h,u,v in zip(hdr,units,vals):
    if h in want: print(f"{h:70s} {u:10s} {v}")
st=[]
for h,u,v in zip(hdr,units,vals):
    if h.startswith('smsp__average_warps_issue_stalled_') and h.endswith('_per_issue_active.ratio'):
        try: st.append((float(v),h[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]))
        except: pass
print("stalls per issue:", ", ".join(f"{n}={v:.2f}" for v,n in sorted(st,reverse=True)[:10]))
