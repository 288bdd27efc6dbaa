"""Per-launch table from an `ncu --metrics ... --csv --log-file` capture (one row per
kernel launch, the metrics as columns).  Usage: python tools/ncu_metrics_table.py CSV [skip]"""
import csv
import sys


def main(path, skip=0):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ik, im, iu, iv, iid = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
    launches = {}
    order = []
    for r in rows[1:]:
        key = r[iid]
        if key not in launches:
            launches[key] = {"name": r[ik]}
            order.append(key)
        launches[key][r[im]] = (r[iv], r[iu])
    cols = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors.sum",
            "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "l1tex__t_sector_hit_rate.pct", "launch__grid_size", "launch__registers_per_thread"]
    short = ["time", "dram_rd", "dram_wr", "lts_sect", "l2hit%", "lts%", "warps%", "issue%", "l1hit%", "grid", "regs"]
    print("| kernel | " + " | ".join(short) + " |")
    print("|---" * (len(short) + 1) + "|")
    for key in order[int(skip):]:
        L = launches[key]
        nm = L["name"].split("(")[0].replace("void ", "")[:40]
        vals = []
        for c in cols:
            v, u = L.get(c, ("", ""))
            vals.append(f"{v} {u}".strip())
        print(f"| {nm} | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    main(*sys.argv[1:])
