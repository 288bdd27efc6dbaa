"""profiles/ncu_traffic.json from an `ncu --set full` report of tools/prof_run.py:
dram read+write bytes and duration per launch of the primal step (K1) and of the
whole dual step (K2 = every kernel from the one after K1 through k_finish<EpiDual>:
k_csrw segments, k_dense, k_finish), keyed by the solver's kernel names (bench.py
`roofline.traffic`).  Usage: python tools/ncu_traffic.py REPORT CONFIG [OUT] [SOURCE_HASH]"""
import csv
import json
import os
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9}


def main(rep, config, out="profiles/ncu_traffic.json", src_hash=None):
    """src_hash: the benchmarked sources' hash (bench.py roofline.traffic_source) when
    the report was captured on a snapshot older than the working tree."""
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    ik = hdr.index("Kernel Name")
    cols = {k: hdr.index(k) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum")}

    def val(r, k):
        return float(r[cols[k]].replace(",", "")) * SCALE.get(units[cols[k]], 1.0)

    groups = {"primal_step_AT": [], "primal_step_AT:corner": [], "dual_step_A": []}
    cur = None
    for r in rows[2:]:
        name = r[ik]
        b = val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
        t = val(r, "gpu__time_duration.sum")
        short = name.split("(")[0]
        if "EpiPrimalT" in name:
            key = "primal_step_AT:corner" if "(bool)1" in name or "EpiPrimalT<1>" in name else "primal_step_AT"
            groups[key].append({"bytes": b, "s": t, "kernels": [short]})
            cur = {"bytes": 0.0, "s": 0.0, "kernels": []}
            continue
        if cur is not None:
            cur["bytes"] += b
            cur["s"] += t
            cur["kernels"].append(short)
            if "k_finish" in name and "EpiDual" in name:
                groups["dual_step_A"].append(cur)
                cur = None
    data = json.load(open(out)) if os.path.exists(out) else {}
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2511_13894_b200 import _build
    data[config] = {"source_hash": src_hash or _build.source_hash()}
    for k, g in groups.items():
        if not g:
            continue
        data[config][k] = {"dram_bytes_per_launch": sum(x["bytes"] for x in g) / len(g),
                           "ncu_seconds_per_launch": sum(x["s"] for x in g) / len(g),
                           "launches_captured": len(g), "kernels": g[-1]["kernels"],
                           "report": os.path.basename(rep)}
    json.dump(data, open(out, "w"), indent=1)
    print(json.dumps(data[config], indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
