"""Aggregate an ncu `--page source --csv --print-source cuda,sass` export by CUDA
source line: warp-stall samples and executed instructions (top N lines)."""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    samp = collections.Counter()
    inst = collections.Counter()
    text = {}
    f = None
    cur = None
    hdr = None
    for row in csv.reader(open(path)):
        if not row:
            continue
        if row[0] == "File Path":
            f = row[1].split("/")[-1]
            continue
        if row[0] == "Line No":
            hdr = row
            continue
        if row[0] == "Function Name" or hdr is None:
            continue
        if row[0]:
            cur = (f, int(row[0]))
            text[cur] = row[1].strip()[:90]
            continue
        try:
            samp[cur] += float(row[4] or 0)
            inst[cur] += float(row[7] or 0)
        except (ValueError, IndexError):
            pass
    tot = sum(samp.values()) or 1
    print(f"total samples {tot:.0f}, instructions {sum(inst.values()):.0f}")
    for k, v in samp.most_common(top):
        print(f"{100 * v / tot:5.1f}% {inst[k]:10.0f}  {k[0]}:{k[1]:<5d} {text.get(k, '')}")


if __name__ == "__main__":
    main()
