"""Brief of an ncu report (raw page): time, DRAM bytes, instructions, pipes, smem, stalls."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines())); h = r[0]
for row in r[2:]:
    print("==", row[h.index("Kernel Name")][:70])
    for k, x in zip(h, row):
        if k in ('gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'smsp__inst_executed.sum',
                 'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
                 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum',
                 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed',
                 'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
                 'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread', 'launch__grid_size',
                 'launch__block_size', 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):
            print(" ", k, x)
        elif k.startswith('smsp__average_warps_issue_stalled_') and k.endswith('_per_issue_active.ratio') and float(x or 0) > 0.15:
            print(" ", k.replace('smsp__average_warps_issue_stalled_', 'stall_').replace('_per_issue_active.ratio', ''), x)
