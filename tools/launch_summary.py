"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

    python tools/launch_summary.py gpurun_out/launches.csv [top]
"""
import collections
import csv
import re
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    h = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[h]
    ki, ui, vi = hdr.index("Kernel Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    out = []
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki]
        m = re.search(r"(\w+)(<[^()]*>)?\(", name)
        short = (m.group(1) + (m.group(2) or "")) if m else name[:40]
        out.append((short, float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)))
    return out


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    tot, cnt = collections.Counter(), collections.Counter()
    for name, us in load(path):
        tot[name] += us
        cnt[name] += 1
    T = sum(tot.values())
    print(f"{'kernel':44s} {'launches':>8s} {'total ms':>10s} {'share':>6s} {'avg us':>9s}")
    for k, v in tot.most_common(top):
        print(f"{k[:44]:44s} {cnt[k]:8d} {v / 1e3:10.3f} {100 * v / T:5.1f}% {v / cnt[k]:9.1f}")
    print(f"total {T / 1e3:.3f} ms over {sum(cnt.values())} launches")


if __name__ == "__main__":
    main()
