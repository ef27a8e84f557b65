"""Summarise an ncu report: key throughput/occupancy metrics, stall reasons,
and the hottest SASS address blocks.  usage: ncu_summary.py report.ncu-rep"""
import csv, subprocess, sys, io

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, u, v = r[0], r[1], r[2]
keys = ['Kernel Name', 'gpu__time_duration.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'lts__t_sector_hit_rate.pct', 'launch__registers_per_thread', 'launch__grid_size', 'launch__block_size']
for k in keys:
    if k in h:
        i = h.index(k)
        print(f"{k:70s} {u[i]:>12s} {v[i]}")
st = [(h[i], v[i]) for i in range(len(h)) if h[i].startswith('smsp__pcsamp_warps_issue_stalled')
      and not h[i].endswith('not_issued')]
st = [(k, float(x.replace(',', ''))) for k, x in st if x not in ('', 'n/a')]
tot = sum(x for _, x in st) or 1
for k, x in sorted(st, key=lambda t: -t[1])[:10]:
    print(f"  stall {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {100 * x / tot:5.1f}%")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(src)))
hh = r[1]
ie, ws = hh.index('Instructions Executed'), hh.index('Warp Stall Sampling (All Samples)')
rows = []
for k, row in enumerate(r[2:]):
    try:
        rows.append((k, float(row[ie] or 0), float(row[ws] or 0), row[1]))
    except (ValueError, IndexError):
        pass
ti = sum(x[1] for x in rows) or 1
tw = sum(x[2] for x in rows) or 1
ops = {}
for _, a, w, s in rows:
    op = s.split()[0] if s.split() else '?'
    if op.startswith('@'):
        op = s.split()[1]
    op = op.split('.')[0]
    o = ops.setdefault(op, [0, 0])
    o[0] += a
    o[1] += w
print("top opcodes (inst%, stall%):")
for op, (a, w) in sorted(ops.items(), key=lambda t: -t[1][0])[:16]:
    print(f"  {op:12s} {100 * a / ti:5.1f}% {100 * w / tw:5.1f}%")
