"""Summarise an ncu report: key metrics per kernel + SASS opcode mix (tools/ncu_summary.py rep [regex])."""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
rx = sys.argv[2] if len(sys.argv) > 2 else "."
M = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'smsp__inst_executed.sum',
     'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed',
     'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
     'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum',
     'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread', 'launch__grid_size']
ST = ['barrier', 'long_scoreboard', 'short_scoreboard', 'wait', 'math_pipe_throttle', 'mio_throttle', 'not_selected',
      'dispatch_stall', 'no_instruction', 'branch_resolving', 'lg_throttle', 'selected']
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h = r[0]
import re
for row in r[2:]:
    name = row[h.index('Kernel Name')]
    if not re.search(rx, name):
        continue
    print(f"== {name[:70]}")
    out = []
    for m in M:
        if m in h:
            out.append(f"{m.split('.')[0].replace('__', ':')}={row[h.index(m)]}")
    print('   ' + '  '.join(out))
    st = []
    for s in ST:
        m = f'smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio'
        if m in h:
            st.append(f"{s}={float(row[h.index(m)]):.2f}")
    print('   stalls/issue: ' + ' '.join(st))
