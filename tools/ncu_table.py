"""Roofline table from ncu --page raw --csv exports (tools/ncu_kernels.sh).

    python tools/ncu_table.py gpurun_out/ncu/*.csv
"""
import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def peak_gbs():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__registers_per_thread"]


def conv(v, unit):
    v = float(v.replace(",", ""))
    scale = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6,
             "ms": 1e-3, "s": 1.0, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    return v * scale.get(unit, 1.0)


def rows(path):
    r = list(csv.reader(open(path)))
    if len(r) < 3:
        return []
    h, u = r[0], r[1]
    out = []
    for row in r[2:]:
        d = {"file": os.path.basename(path)}
        name = row[h.index("Kernel Name")]
        m = re.search(r"(\w+)(<[^()]*>)?\(", name)
        d["kernel"] = (m.group(1) + (m.group(2) or "")) if m else name[:40]
        for w in WANT:
            if w in h:
                i = h.index(w)
                try:
                    d[w] = conv(row[i], u[i])
                except ValueError:
                    d[w] = None
        out.append(d)
    return out


def main():
    peak, src = peak_gbs()
    print(f"| kernel | config | duration us | DRAM MB (r+w) | DRAM GB/s | of HBM peak ({src} {peak:.0f}) | SM busy % | warps active % | DMMA pipe % |")
    print("|---|---|---|---|---|---|---|---|---|")
    for p in sys.argv[1:]:
        for d in rows(p):
            t = d.get("gpu__time_duration.sum") or 0
            by = (d.get("dram__bytes_read.sum") or 0) + (d.get("dram__bytes_write.sum") or 0)
            gbs = by / t / 1e9 if t else 0
            dm = d.get("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active")
            print(f"| {d['kernel']} | {d['file'][:-4]} | {t*1e6:.1f} | {by/1e6:.2f} | {gbs:.0f} | {gbs/peak:.3f} | "
                  f"{(d.get('sm__throughput.avg.pct_of_peak_sustained_elapsed') or 0):.1f} | "
                  f"{(d.get('sm__warps_active.avg.pct_of_peak_sustained_active') or 0):.1f} | "
                  f"{'' if dm is None else f'{dm:.1f}'} |")


if __name__ == "__main__":
    main()
