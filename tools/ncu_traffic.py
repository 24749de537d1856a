"""DRAM traffic per sweep pair from an ncu --set full capture (raw CSV), for the
bench roofline's `traffic` key: python tools/ncu_traffic.py <raw.csv> <config> [out.json]

The capture holds consecutive launches of one refinement step's sweep kernels;
each kernel's first launch is counted once (one forward+backward pair)."""
import csv
import json
import os
import re
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main():
    path, config = sys.argv[1], sys.argv[2]
    out = sys.argv[3] if len(sys.argv) > 3 else None
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    ri, wi = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    ti = hdr.index("gpu__time_duration.sum")
    seen = {}
    for r in rows[2:]:
        m = re.search(r"(\w+)<", r[ki]) or re.search(r"(\w+)\(", r[ki])
        name = m.group(1) if m else r[ki][:30]
        if name in seen:
            continue
        rd = float(r[ri].replace(",", "")) * SCALE.get(units[ri], 1)
        wr = float(r[wi].replace(",", "")) * SCALE.get(units[wi], 1)
        seen[name] = {"dram_read": rd, "dram_write": wr, "us": float(r[ti].replace(",", "")) *
                      (1e-3 if units[ti].startswith("n") else 1.0)}
    total = sum(v["dram_read"] + v["dram_write"] for v in seen.values())
    doc = {"bytes": total, "source": f"ncu --set full, one launch of each sweep kernel of a {config} refinement "
                                     f"step ({os.path.basename(path)})", "per_kernel": seen}
    print(json.dumps(doc, indent=1))
    if out:
        full = json.load(open(out)) if os.path.exists(out) else {}
        full[config] = doc
        json.dump(full, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
