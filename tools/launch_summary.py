"""Per-kernel totals of an ncu launch list (gpu__time_duration.sum CSV).

    python tools/launch_summary.py launches.csv [steps]
"""
import collections
import csv
import re
import sys


def short(name):
    n = re.sub(r"\(.*$", "", name.replace("(anonymous namespace)", "").replace("<unnamed>", ""))
    n = re.sub(r"<.*$", "", n)
    return n.split("::")[-1]


def main():
    path = sys.argv[1]
    steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, mi = h.index("Kernel Name"), h.index("Metric Value")
    agg, cnt = collections.defaultdict(float), collections.Counter()
    for r in data:
        n = short(r[ki])
        agg[n] += float(r[mi].replace(",", "")) / 1e3
        cnt[n] += 1
    tot = sum(agg.values())
    print(f"launches {len(data)}, {tot / steps:.1f} us per step ({steps:g} steps)")
    for k, v in sorted(agg.items(), key=lambda x: -x[1]):
        print(f"{v / steps:9.1f} us/step  {cnt[k] / steps:5.1f} launches/step  {100 * v / tot:5.1f}%  {k}")


if __name__ == "__main__":
    main()
