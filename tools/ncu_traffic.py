"""profiles/ncu_traffic.json from an `ncu --set full` report: dram read+write bytes
per launch of each hot kernel, keyed by the solver's kernel names (bench.py
`roofline.traffic`).  Usage: python tools/ncu_traffic.py REPORT CONFIG [OUT]"""
import csv
import json
import os
import subprocess
import sys

# ncu kernel (demangled, template args) -> solver kernel-time name
MAP = [("EpiPrimalT<0>", "primal_step_AT"), ("EpiPrimalT<1>", "primal_step_AT:corner"),
       ("EpiDual", "dual_step_A"), ("EpiCheckN", "check_eval_AT"), ("EpiCheckM", "check_eval_A")]


def main(rep, config, out="profiles/ncu_traffic.json"):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr = rows[0]
    ik, ir, iw, it = (hdr.index("Kernel Name"), hdr.index("dram__bytes_read.sum"),
                      hdr.index("dram__bytes_write.sum"), hdr.index("gpu__time_duration.sum"))
    units = rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    per = {}
    for r in rows[2:]:
        name = r[ik]
        key = next((v for k, v in MAP if k.replace("<0>", "<(bool)0>").replace("<1>", "<(bool)1>") in name
                    or k in name), None)
        if key is None:
            continue
        b = float(r[ir].replace(",", "")) * scale[units[ir]] + float(r[iw].replace(",", "")) * scale[units[iw]]
        d = per.setdefault(key, {"launches": 0, "dram_bytes": 0.0, "kernels": set()})
        d["launches"] += 1 if "k_finish" not in name else 0
        d["dram_bytes"] += b
        d["kernels"].add(name.split("(")[0][:80])
    data = json.load(open(out)) if os.path.exists(out) else {}
    data[config] = {k: {"dram_bytes_per_launch": v["dram_bytes"] / max(v["launches"], 1),
                        "kernels": sorted(v["kernels"]), "report": os.path.basename(rep)}
                    for k, v in per.items()}
    json.dump(data, open(out, "w"), indent=1)
    print(json.dumps(data[config], indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
