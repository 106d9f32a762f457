"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per kernel count, total device time and share."""
import collections
import csv
import sys


def summarise(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    i_name, i_val = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        short = r[i_name].split("(")[0].replace("void ", "")[:70]
        agg[short][0] += 1
        agg[short][1] += float(r[i_val].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    out = []
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| {k} | {c} | {t / 1e3:.1f} | {t / tot:.1%} | {t / c / 1e3:.2f} |")
    return ["| kernel | launches | total us | share | avg us |", "|---|---|---|---|---|"] + out


if __name__ == "__main__":
    print("\n".join(summarise(sys.argv[1])))
