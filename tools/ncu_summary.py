"""Summarise an ncu report: per-kernel metrics and top SASS stall lines."""
import csv
import subprocess
import sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_sector_hit_rate.pct',
        'l1tex__t_sector_hit_rate.pct', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__grid_size', 'smsp__inst_executed.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__average_warp_latency_per_inst_issued.ratio']


def raw(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {'kernel': r[hdr.index('Kernel Name')][:60]}
        for w in WANT:
            if w in hdr:
                d[w] = (r[hdr.index(w)], units[hdr.index(w)])
        res.append(d)
    return res


def stalls(rep, match, top=15):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                         capture_output=True, text=True).stdout.split('\n')
    starts = [i for i, l in enumerate(out) if l.startswith('"Kernel Name"')] + [len(out)]
    for a, b in zip(starts, starts[1:]):
        if match not in out[a]:
            continue
        rows = list(csv.reader(out[a + 1:b]))
        hdr = rows[0]
        ix, isrc, ist = hdr.index('Instructions Executed'), hdr.index('Source'), hdr.index('Warp Stall Sampling (All Samples)')
        data = [r for r in rows[1:] if len(r) == len(hdr)]
        tot = sum(float(r[ist] or 0) for r in data)
        print(f"{out[a][:100]}\n  stall samples {tot:.0f}, instructions {sum(float(r[ix] or 0) for r in data):.3g}")
        for r in sorted(data, key=lambda r: -float(r[ist] or 0))[:top]:
            print(f"  {float(r[ist] or 0) / tot * 100:5.1f}% {float(r[ix] or 0):>11.0f} {r[isrc][:80]}")
        return


if __name__ == '__main__':
    rep = sys.argv[1]
    for d in raw(rep):
        print(d['kernel'])
        for k, v in d.items():
            if k != 'kernel':
                print(f"   {k:60s} {v[0]} {v[1]}")
    for m in sys.argv[2:]:
        stalls(rep, m)
