"""Per-region instruction / stall shares of one kernel in an ncu report (SASS page)."""
import csv
import subprocess
import sys

rep, match = sys.argv[1], sys.argv[2]
lines = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                       capture_output=True, text=True).stdout.split('\n')
starts = [i for i, l in enumerate(lines) if l.startswith('"Kernel Name"')] + [len(lines)]
for a, b in zip(starts, starts[1:]):
    if match not in lines[a]:
        continue
    rows = list(csv.reader(lines[a + 1:b]))
    hdr = rows[0]
    ix, isrc, ist = hdr.index('Instructions Executed'), hdr.index('Source'), hdr.index('Warp Stall Sampling (All Samples)')
    data = [r for r in rows[1:] if len(r) == len(hdr)]
    vals = [float(r[ix] or 0) for r in data]
    stl = [float(r[ist] or 0) for r in data]
    tot, stot = sum(vals), sum(stl)
    print(lines[a][:110], '\n total inst', tot, 'stall samples', stot)
    i = 0
    while i < len(data):
        if vals[i] == 0:
            i += 1
            continue
        j = i
        while j < len(data) and vals[j] > 0 and abs(vals[j] - vals[i]) < 0.05 * vals[i] + 1:
            j += 1
        sh, ss = sum(vals[i:j]) / tot * 100, sum(stl[i:j]) / stot * 100
        if sh > 1.5 or ss > 2:
            print(f"{i:5d}-{j:5d} inst {sh:5.1f}% stall {ss:5.1f}% count={vals[i]:.0f} n={j - i} :: "
                  f"{data[i][isrc][:38]} ... {data[j - 1][isrc][:38]}")
            if len(sys.argv) > 3:
                for k in range(i, j):
                    if stl[k] > 0.01 * stot:
                        print(f"        {stl[k] / stot * 100:5.1f}% {data[k][isrc][:70]}")
        i = max(j, i + 1)
    break
