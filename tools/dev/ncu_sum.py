"""Summarise an `ncu --page raw --csv` export (dev): time, DRAM bytes,
instructions, issue, occupancy and the top stall reasons per kernel."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[0]
want = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'smsp__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__grid_size', 'launch__block_size']
stalls = [(h[i], i) for i in range(len(h)) if h[i].startswith('smsp__pcsamp_warps_issue_stalled_')
          and not h[i].endswith('not_issued')]
for r in rows[2:]:
    print('---')
    for w in want:
        if w in h:
            print(f'{w:60s} {r[h.index(w)]}')
    tot = sum(float(r[i] or 0) for _, i in stalls) or 1.0
    top = sorted(((float(r[i] or 0) / tot * 100, n.replace('smsp__pcsamp_warps_issue_stalled_', ''))
                  for n, i in stalls), reverse=True)[:7]
    print('stalls:', ', '.join(f'{n} {v:.1f}%' for v, n in top))
