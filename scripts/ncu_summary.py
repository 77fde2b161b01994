"""Summarise an ncu report (raw metrics + hottest SASS blocks) — run in the build container."""
import csv, io, subprocess, sys

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))

KEYS = ['gpu__time_duration.sum', 'launch__grid_size', 'launch__block_size', 'launch__registers_per_thread',
        'smsp__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum',
        'l1tex__throughput.avg.pct_of_peak_sustained_active', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__cycles_elapsed.avg']

def hot(rep, n=20):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]; data = rows[2:]
    isrc = h.index('Source'); ist = h.index('Warp Stall Sampling (All Samples)'); iex = h.index('Instructions Executed')
    tot = sum(int(r[iex]) for r in data if r[iex].isdigit()) or 1
    totst = sum(int(r[ist]) for r in data if r[ist].isdigit()) or 1
    blocks = []; cur = None
    for idx, r in enumerate(data):
        ex = int(r[iex]) if r[iex].isdigit() else 0; st = int(r[ist]) if r[ist].isdigit() else 0
        if cur is None or ex != cur['ex']:
            cur = {'start': idx, 'ex': ex, 'n': 0, 'st': 0, 'ops': []}; blocks.append(cur)
        cur['n'] += 1; cur['st'] += st; cur['ops'].append(r[isrc].split()[0] if r[isrc].split() else '')
    blocks.sort(key=lambda b: -b['ex'] * b['n'])
    lines = []
    for b in blocks[:n]:
        lines.append(f"@{b['start']:5d} n={b['n']:3d} exec={b['ex']:9d} inst-share={b['ex']*b['n']/tot*100:5.1f}% "
                     f"stall-share={b['st']/totst*100:5.1f}% {' '.join(b['ops'][:12])}")
    return lines

if __name__ == "__main__":
    for rep in sys.argv[1:]:
        v, u = raw(rep)
        print("==", rep)
        for k in KEYS:
            if k in v: print(f"  {k:70s} {v[k]:>18s} {u.get(k,'')}")
        for k in sorted(v):
            if k.startswith('smsp__average_warps_issue_stalled_') and k.endswith('_per_issue_active.ratio'):
                try:
                    if float(v[k]) > 0.15: print(f"  {k:70s} {v[k]:>18s}")
                except ValueError: pass
        for l in hot(rep): print("  ", l)
