"""profiles/traffic.json from an `ncu --set full` raw CSV: median DRAM bytes
(read + write) per launch of each kernel, under the names bench.py's
roofline uses.  The median is the steady iteration: a solve's first pv pass
(no p / v to read) and its tail (converged components skipped) move less.
Usage: python tools/traffic_from_ncu.py raw.csv config"""
import csv
import json
import os
import re
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def bench_names(kernel):
    k = re.sub(r"^void ", "", kernel)
    base = re.match(r"(?:pf::)?(\w+)", k).group(1)
    if base == "k_bi_tiled":
        m = re.search(r"k_bi_tiled<(\w+),\s*(\d)", k)
        adj = m.group(1) in ("1", "true")
        nm = {"0": "k_bi_pv", "1": "k_bi_st", "2": "k_bi_init",
              "3": "k_bi_verify"}[m.group(2)]
        return [nm + (" (adjoint)" if adj else "")]
    if base in ("k_bi_pv", "k_bi_st"):
        adj = re.search(r",\s*(?:true|1)>", k) is not None
        return [base + (" (adjoint)" if adj else "")]
    if base == "k_bi_xr":
        return ["k_bi_xr", "k_bi_xr (adjoint)"]
    return [base]


def main(path, config):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    acc = defaultdict(list)
    for r in rows[2:]:
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            b += float(r[idx[m]].replace(",", "")) * scale[units[idx[m]]]
        for nm in bench_names(r[idx["Kernel Name"]]):
            acc[nm].append(b)
    out_path = os.path.join(ROOT, "profiles", "traffic.json")
    data = json.load(open(out_path)) if os.path.exists(out_path) else {}
    data.setdefault(config, {}).update(
        {k: sorted(v)[len(v) // 2] for k, v in acc.items()})
    data["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch "
                     "(median over the step's launches) from ncu --set full "
                     "(tools/traffic_from_ncu.py)")
    json.dump(data, open(out_path, "w"), indent=1, sort_keys=True)
    print(json.dumps(data[config], indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
