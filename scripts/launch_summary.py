"""Aggregates an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel.
Usage: python scripts/launch_summary.py launches.csv [--grid] [--top N]"""
import collections
import csv
import sys


def main(path, by_grid=False, top=15):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ik, iv, ig = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Grid Size")
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        name = r[ik].split("(")[0].replace("void ", "").replace("tgk::<unnamed>::", "").replace("tgk::", "")
        key = (name, r[ig]) if by_grid else (name, "")
        agg[key].append(float(r[iv].replace(",", "")) / 1e3)
    tot = sum(sum(v) for v in agg.values())
    n = sum(len(v) for v in agg.values())
    print(f"total {tot / 1e3:.2f} ms over {n} launches")
    for (k, g), v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))[:top]:
        print(f"{k:38s} {g:16s} n={len(v):6d} {sum(v) / 1e3:9.2f} ms {sum(v) / tot * 100:5.1f}%  mean {sum(v) / len(v):8.1f} us")


if __name__ == "__main__":
    a = sys.argv[1:]
    top = int(a[a.index("--top") + 1]) if "--top" in a else 15
    main(a[0], "--grid" in a, top)
