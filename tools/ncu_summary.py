"""Summarise an ncu report (details + a few raw metrics) per kernel."""
import csv
import subprocess
import sys

rep = sys.argv[1]
want = ['Duration', 'DRAM Throughput', 'L1/TEX Hit Rate', 'L2 Hit Rate', 'Compute (SM) Throughput',
        'Memory Throughput', 'Achieved Occupancy', 'Registers Per Thread', 'Executed Ipc Active',
        'Issue Slots Busy', 'L1/TEX Cache Throughput', 'L2 Cache Throughput',
        'Theoretical Occupancy', 'Warp Cycles Per Issued Instruction', 'No Eligible',
        'Eligible Warps Per Scheduler']
out = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
ki, mi, vi, ui = (hdr.index(k) for k in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit'))
for r in rows[1:]:
    if r[mi] in want:
        print(f"{r[ki][:28]:28s} | {r[mi]:36s} {r[vi]} {r[ui]}")
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr = rows[0]
keys = ['dram__bytes_read.sum', 'dram__bytes_write.sum', 'l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum',
        'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum', 'smsp__inst_executed.sum',
        'l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_elapsed',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active']
for r in rows[2:]:
    name = r[hdr.index('Kernel Name')][:28]
    print(name, {k.split('.')[0].replace('l1tex__', '').replace('pipe_lsu_mem_', ''): r[hdr.index(k)]
                 for k in keys if k in hdr})
